"""Run torch SDPA (vendor kernel) on one config for ncu inspection (tuning aid).
usage: python scripts/vendor_probe.py B H S D [iters]"""
import sys
import torch
B, H, S, D = (int(x) for x in sys.argv[1:5])
n = int(sys.argv[5]) if len(sys.argv) > 5 else 3
q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(n):
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
print("ok", o.shape)
