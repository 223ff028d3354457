set -u
O=gpurun_out/sanitize2; mkdir -p $O; : > $O/summary.txt
for tool in racecheck memcheck; do
  for d in 64 128 256; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 --log-file $O/${tool}_D$d.log python scripts/sanitize.py --quick $d > $O/${tool}_D$d.out 2>&1
    echo "$tool D=$d rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${tool}_D$d.log | tail -1 | sed 's/=========//') | $(tail -1 $O/${tool}_D$d.out)" >> $O/summary.txt
  done
done
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
cat $O/summary.txt; tail -2 $O/pytest_gpu.txt
