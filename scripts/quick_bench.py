"""Quick device-timed sweep of a few configs (tuning aid; not the contract bench).
usage: python scripts/quick_bench.py [--torch] [--long]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2603_01960_b200 as ta

cfgs = [(1, 8, 512, 64, torch.float16), (4, 16, 4096, 64, torch.bfloat16),
        (8, 32, 4096, 128, torch.bfloat16), (1, 16, 16384, 128, torch.bfloat16)]
if "--long" in sys.argv:
    cfgs.append((8, 8, 32768, 128, torch.bfloat16))
for (B, H, S, D, dt) in cfgs:
    q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=dt) for _ in range(3))
    o = torch.empty_like(q)
    for _ in range(3):
        ta.sdpa(q, k, v, out=o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        ta.sdpa(q, k, v, out=o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = 4 * B * H * S * S * D
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v)
    err = (o.float() - ref.float()).abs().max().item()
    line = f"B{B} H{H} S{S} D{D} {str(dt)[6:]}: {ms:.3f} ms {fl / ms / 1e9:7.1f} TFLOP/s maxdiff {err:.2e}"
    if "--torch" in sys.argv:
        e0.record()
        for _ in range(n):
            torch.nn.functional.scaled_dot_product_attention(q, k, v)
        e1.record()
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1) / n
        line += f" | torch sdpa {ms2:.3f} ms {fl / ms2 / 1e9:7.1f} TFLOP/s"
    print(line, flush=True)
