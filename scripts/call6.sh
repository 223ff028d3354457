set -u
O=gpurun_out/c6; mkdir -p $O
L=paper_2603_01960_b200/_lib
TILEATTN_B200_LIB=$L/var/lib_d64split.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "64 or cfg1 or golden or random or causal or padding" > $O/pytest_d64split.txt 2>&1; echo "rc=$?" >> $O/pytest_d64split.txt; tail -3 $O/pytest_d64split.txt
timeout 1200 python scripts/ab.py --reps 2 64,16,1024,64 4,16,8192,64 4,16,1024,64 8,32,4096,64,f16 -- $L/libtileattn_b200.so $L/var/lib_d64split.so $L/var/lib_d64pp.so > $O/ab.txt 2>&1
cat $O/ab.txt
bash scripts/sanitize.sh
mkdir -p gpurun_out/sanitize_obs
for d in 64 128 160 256; do
  TILEATTN_B200_LIB=$L/var/lib_observe.so timeout 900 compute-sanitizer --tool synccheck --print-limit 50 \
    --log-file gpurun_out/sanitize_obs/synccheck_D$d.log python scripts/sanitize.py $d > gpurun_out/sanitize_obs/synccheck_D$d.out 2>&1
  echo "synccheck(observe build) D=$d rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize_obs/synccheck_D$d.log | tail -1 | sed 's/=========//') | $(tail -1 gpurun_out/sanitize_obs/synccheck_D$d.out)" >> gpurun_out/sanitize_obs/summary.txt
done
cat gpurun_out/sanitize_obs/summary.txt
