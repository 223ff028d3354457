set -u
O=gpurun_out/c11; mkdir -p $O
L=paper_2603_01960_b200/_lib
timeout 120 python scripts/probe.py 64 32 8 > $O/probe.txt 2>&1; echo "rc=$?" >> $O/probe.txt
tail -3 $O/probe.txt
if grep -q "failures: 0" $O/probe.txt; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.txt 2>&1; echo "rc=$?" >> $O/pytest_parity.txt; tail -3 $O/pytest_parity.txt
  timeout 900 python scripts/ab.py --reps 2 64,16,1024,64 4,16,1024,64 4,16,4096,64 4,16,16384,64 8,32,4096,64,f16 1,8,512,64,f16 -- $L/libtileattn_b200.so $L/var/lib_nopersist.so > $O/ab.txt 2>&1
  cat $O/ab.txt
fi
