# One GPU evidence pass (run under gpurun from the repo root):
#   parity tests, smoke, contract bench, sweep vs vendor, ncu launch list and
#   one ncu --set full capture of the bench kernel.  Outputs: gpurun_out/round/
set -u
O=gpurun_out/round
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench_n1.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; tail -1 $O/bench_ref.log > $O/bench_ref.json
timeout 1200 python bench.py --sweep --vendor > $O/sweep.log 2>&1; grep '^{' $O/sweep.log > $O/sweep.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sdpa_fwd_kernel -s 3 -c 1 \
  -o $O/prof_long python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
ls -la $O
