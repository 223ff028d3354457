# A/B run of kernel variants on the GPU box: parity tests + quick bench + trace
# usage: bash scripts/gpu_ab.sh "<variants>"
mkdir -p gpurun_out
for V in $1; do
  echo "=== variant $V"
  TILEATTN_B200_VARIANT=$V timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
  TILEATTN_B200_VARIANT=$V timeout 300 python scripts/quick_bench.py --long 2>&1
  TILEATTN_B200_VARIANT=$V timeout 120 python scripts/trace_timeline.py 1 16 16384 128 2>&1 | sed -n '1,8p;/mean over/,$p'
done
