set -u
O=gpurun_out/c4; mkdir -p $O
L=paper_2603_01960_b200/_lib
timeout 900 python scripts/ab.py --reps 2 8,64,32768,128 64,16,1024,64 -- $L/libtileattn_b200.so $L/var/lib_halfkv.so $L/var/lib_split.so > $O/ab.txt 2>&1
cat $O/ab.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.txt 2>&1; echo "rc=$?" >> $O/pytest_parity.txt; tail -3 $O/pytest_parity.txt
