set -u
O=gpurun_out/c27; mkdir -p $O
timeout 300 python scripts/stress_bn64.py 300 130 f16 > $O/plain.txt 2>&1; tail -3 $O/plain.txt
timeout 300 python scripts/stress_bn64.py 300 700 bf16 > $O/plain2.txt 2>&1; tail -3 $O/plain2.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python scripts/stress_bn64.py 20 130 f16 > $O/memcheck.txt 2>&1; tail -8 $O/memcheck.txt
