set -u
O=gpurun_out/c29; mkdir -p $O
for i in 1 2 3 4; do timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python scripts/sanitize.py --quick 128 > $O/memcheck_$i.txt 2>&1; echo "run $i: $(grep -c FAIL $O/memcheck_$i.txt) FAIL, $(grep 'ERROR SUMMARY' $O/memcheck_$i.txt)"; done
timeout 300 python scripts/stress_bn64.py 300 130 f16 | tail -1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt; tail -2 $O/pytest_gpu.txt
