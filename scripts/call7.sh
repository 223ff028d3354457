set -u
O=gpurun_out/c7; mkdir -p $O
L=paper_2603_01960_b200/_lib
TILEATTN_B200_LIB=$L/var/lib_pair.so timeout 120 python scripts/probe.py 128 96 > $O/probe_pair.txt 2>&1; echo "rc=$?" >> $O/probe_pair.txt
cat $O/probe_pair.txt
if grep -q "failures: 0" $O/probe_pair.txt; then
  timeout 600 python scripts/ab.py --reps 2 8,64,32768,128 8,32,4096,128 4,16,1024,128 -- $L/libtileattn_b200.so $L/var/lib_pair.so > $O/ab.txt 2>&1
  cat $O/ab.txt
fi
TILEATTN_B200_LIB=$L/var/lib_nostore.so timeout 600 compute-sanitizer --tool initcheck --print-limit 20 --log-file $O/initcheck_nostore_D64.log python scripts/sanitize.py --quick 64 > $O/initcheck_nostore_D64.out 2>&1
grep "ERROR SUMMARY" $O/initcheck_nostore_D64.log
