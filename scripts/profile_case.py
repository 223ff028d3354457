"""Run one SDPA config a few times (target for ncu captures).
usage: python scripts/profile_case.py B H S D dtype [iters]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2603_01960_b200 as ta

B, H, S, D = (int(x) for x in sys.argv[1:5])
dt = {"bf16": torch.bfloat16, "f16": torch.float16}[sys.argv[5]]
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 3
q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=dt) for _ in range(3))
o = torch.empty_like(q)
for _ in range(iters):
    ta.sdpa(q, k, v, out=o)
torch.cuda.synchronize()
print("done", B, H, S, D, sys.argv[5])
