set -u
O=gpurun_out/c28; mkdir -p $O
for i in 1 2 3; do timeout 300 python scripts/sanitize.py --quick 128 > $O/plain_$i.txt 2>&1; grep -c FAIL $O/plain_$i.txt; grep FAIL $O/plain_$i.txt; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python scripts/sanitize.py --quick 128 > $O/memcheck.txt 2>&1; grep "FAIL\|SUMMARY" $O/memcheck.txt
