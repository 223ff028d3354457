set -u
O=gpurun_out/c8; mkdir -p $O
L=paper_2603_01960_b200/_lib
for lib in libtileattn_b200.so var/lib_pair.so; do
  echo "== $lib" >> $O/trace.txt
  TILEATTN_B200_LIB=$L/$lib timeout 120 python scripts/trace_timeline.py 1 16 16384 128 >> $O/trace.txt 2>&1
done
cat $O/trace.txt | grep -v "^ *[0-9]"
timeout 600 python scripts/ab.py --reps 1 8,64,32768,128 -- $L/libtileattn_b200.so $L/var/lib_pair.so > $O/ab.txt 2>&1
cat $O/ab.txt
