set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
./build/mb_pipes > gpurun_out/mb_pipes.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
timeout 300 python scripts/quick_bench.py --torch --long > gpurun_out/qb_v0.txt 2>&1
TILEATTN_B200_VARIANT=1 timeout 300 python scripts/quick_bench.py --long > gpurun_out/qb_v1.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/mb_pipes.txt gpurun_out/qb_v0.txt gpurun_out/qb_v1.txt
