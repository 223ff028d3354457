# compute-sanitizer over every kernel instantiation (run under gpurun from the
# repo root): one process per tool and head dim, so an error in one kernel
# does not hide the others.  Logs: gpurun_out/sanitize/<tool>_D<d>.log,
# summary: gpurun_out/sanitize/summary.txt.  racecheck / initcheck use the
# quick case list (one ragged shape per mask and dtype).
set -u
O=gpurun_out/sanitize
mkdir -p $O
: > $O/summary.txt
for tool in memcheck synccheck racecheck initcheck; do
  extra=""; quick=""
  [ $tool = racecheck ] && extra="--racecheck-report all" && quick="--quick"
  [ $tool = initcheck ] && quick="--quick"
  for d in 64 128 160 256; do
    timeout 900 compute-sanitizer --tool $tool $extra --print-limit 100 \
      --log-file $O/${tool}_D$d.log python scripts/sanitize.py $quick $d > $O/${tool}_D$d.out 2>&1
    rc=$?
    echo "$tool D=$d rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${tool}_D$d.log | tail -1 | sed 's/=========//') | $(tail -1 $O/${tool}_D$d.out)" >> $O/summary.txt
  done
done
cat $O/summary.txt
