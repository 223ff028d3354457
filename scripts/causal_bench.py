"""Causal vs non-causal timing (report; FLOPs counted as in the reference flop_rate, 4*B*H*S^2*D,
and the causal-effective half of it)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import time
t_start = time.time()
import torch
print(f"[{time.time()-t_start:.1f}s] torch imported", flush=True)
import paper_2603_01960_b200 as ta
for (B, H, S, D) in [(8, 32, 4096, 128), (1, 16, 16384, 128), (4, 16, 8192, 64)]:
    q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    print(f"[{time.time()-t_start:.1f}s] inputs B{B} H{H} S{S} D{D}", flush=True)
    for causal in (False, True):
        for _ in range(3):
            ta.sdpa(q, k, v, causal=causal)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ta.sdpa(q, k, v, causal=causal)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        e0.record()
        for _ in range(10):
            torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)
        e1.record(); torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1) / 10
        fl = 4 * B * H * S * S * D * (0.5 if causal else 1.0)
        print(f"B{B} H{H} S{S} D{D} causal={causal}: {ms:.3f} ms {fl/ms/1e9:7.1f} TF/s (effective) | torch {ms2:.3f} ms {fl/ms2/1e9:7.1f}", flush=True)
