"""Repeat the 64-key split kernel's slow-path case and report mismatches
(race hunting; usage: python scripts/stress_bn64.py [iters] [S] [dtype])."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_01960_b200 as ta  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
S = int(sys.argv[2]) if len(sys.argv) > 2 else 130
dt = torch.float16 if (sys.argv[3] if len(sys.argv) > 3 else "f16") == "f16" else torch.bfloat16
torch.manual_seed(0)
B, H, D = 2, 2, 128
bad = 0
for it in range(iters):
    q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=dt) for _ in range(3))
    o = ta.sdpa(q, k, v, scale=1.0, schedule=ta.TileSchedule(64, 64, 2))
    s = torch.einsum("bhqd,bhkd->bhqk", q.float(), k.float())
    ref = torch.softmax(s, -1) @ v.float()
    err = (o.float() - ref).abs()
    if err.max().item() > 5e-3 * (8 if dt == torch.bfloat16 else 1):
        bad += 1
        idx = (err.amax(-1) > 5e-2).nonzero()
        print(f"iter {it}: max err {err.max().item():.3e}, bad rows {idx[:8].tolist()} ({len(idx)})",
              flush=True)
print(f"{bad} / {iters} bad")
