# round-2 final evidence pass (gpurun from the repo root)
set -u
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
rm -f $O/parity.jsonl
TA_PARITY_OUT=$O/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; cat $O/smoke.txt
timeout 900 python bench.py > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench_n1.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; tail -1 $O/bench_ref.log > $O/bench_ref.json
timeout 1500 python bench.py --sweep --vendor > $O/sweep.log 2>&1; grep '^{' $O/sweep.log > $O/sweep.jsonl
timeout 600 python scripts/tile_table.py $O/tile_table.md > $O/tile_table.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdpa_fwd_kernel -s 3 -c 1 \
  -o $O/prof_long python scripts/profile_case.py 8 64 32768 128 bf16 5 > $O/ncu_long.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdpa_fwd_kernel -s 3 -c 1 \
  -o $O/prof_d256 python scripts/profile_case.py 8 32 4096 256 bf16 5 > $O/ncu_d256.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdpa_fwd_kernel -s 3 -c 1 \
  -o $O/prof_d64 python scripts/profile_case.py 8 32 4096 64 bf16 5 > $O/ncu_d64.log 2>&1
ls -la $O
