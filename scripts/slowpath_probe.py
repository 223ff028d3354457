"""Times a few configs individually (each guarded), for regressions that only hit some CTAs."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2603_01960_b200 as ta
for (B, H, S, D) in [(1, 1, 1024, 128), (1, 16, 1024, 128), (1, 148, 1024, 128), (1, 16, 8192, 128), (2, 16, 4096, 128), (8, 32, 4096, 128)]:
    q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = ta.sdpa(q, k, v); torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(3):
        ta.sdpa(q, k, v, out=o)
    torch.cuda.synchronize()
    ms = (time.time() - t0) / 3 * 1e3
    print(f"B{B} H{H} S{S} D{D}: {ms:.3f} ms  {4*B*H*S*S*D/ms/1e9:.1f} TF/s", flush=True)
