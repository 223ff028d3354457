# compute-sanitizer over every kernel instantiation (run under gpurun from the
# repo root).  Logs: gpurun_out/sanitize/<tool>.log, summary: summary.txt
set -u
O=gpurun_out/sanitize
mkdir -p $O
: > $O/summary.txt
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 200 \
    --log-file $O/$tool.log python scripts/sanitize.py "$@" > $O/$tool.out 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/$tool.log | tail -1) $(tail -1 $O/$tool.out)" >> $O/summary.txt
done
cat $O/summary.txt
