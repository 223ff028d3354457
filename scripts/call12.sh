set -u
O=gpurun_out/c12; mkdir -p $O
L=paper_2603_01960_b200/_lib
timeout 900 python scripts/ab.py --reps 2 64,16,1024,64 4,16,16384,64 -- $L/libtileattn_b200.so $L/var/lib_persist.so $L/var/lib_persist_st1.so $L/var/lib_persist_st3.so > $O/ab.txt 2>&1
cat $O/ab.txt
