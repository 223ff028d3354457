# split-softmax + 64-key tile validation and A/B (gpurun from the repo root)
set -u
O=gpurun_out/c2; mkdir -p $O
L=paper_2603_01960_b200/_lib
timeout 600 python -m pytest tests/test_gpu_parity.py -q > $O/pytest_parity.txt 2>&1; echo "rc=$?" >> $O/pytest_parity.txt
tail -3 $O/pytest_parity.txt
timeout 900 python scripts/ab.py --reps 2 8,64,32768,128 8,32,4096,128 4,16,2048,128,causal -- $L/libtileattn_b200.so $L/var/lib_nosplit.so $L/var/lib_emu0.so $L/var/lib_emu2.so $L/var/lib_emu6.so $L/var/lib_noobs.so > $O/ab.txt 2>&1
cat $O/ab.txt
timeout 300 python scripts/ab.py --tn 64 --reps 1 8,64,32768,128 8,32,4096,128 -- $L/libtileattn_b200.so > $O/ab_bn64.txt 2>&1
cat $O/ab_bn64.txt
timeout 600 python scripts/tile_table.py gpurun_out/c2/tile_table.md > gpurun_out/c2/tile_table.log 2>&1; cat gpurun_out/c2/tile_table.log
