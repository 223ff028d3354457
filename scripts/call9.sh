set -u
O=gpurun_out/c9; mkdir -p $O
L=paper_2603_01960_b200/_lib
TILEATTN_B200_LIB=$L/var/lib_pair.so timeout 120 python scripts/probe.py 128 96 > $O/probe_pair.txt 2>&1; echo "rc=$?" >> $O/probe_pair.txt
tail -2 $O/probe_pair.txt
timeout 600 python scripts/ab.py --reps 2 8,64,32768,128 8,32,4096,128 4,16,1024,128 -- $L/libtileattn_b200.so $L/var/lib_pair.so > $O/ab.txt 2>&1
cat $O/ab.txt
TILEATTN_B200_LIB=$L/var/lib_pair.so timeout 120 python scripts/trace_timeline.py 1 16 16384 128 > $O/trace_pair.txt 2>&1
grep -v "^ *[0-9]" $O/trace_pair.txt
