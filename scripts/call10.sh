set -u
O=gpurun_out/c10; mkdir -p $O
L=paper_2603_01960_b200/_lib
timeout 900 python scripts/ab.py --reps 2 8,64,32768,128 4,16,8192,64 -- $L/libtileattn_b200.so $L/var/lib_noexp.so $L/var/lib_nomma.so $L/var/lib_nomma_noexp.so torch > $O/ab.txt 2>&1
cat $O/ab.txt
