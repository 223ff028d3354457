"""Race hunting on the stale-max slow path: random inputs at scale 1 (scores
8-16x the default, so the O rescale runs on many tiles), repeated, against
torch fp32.  usage: python scripts/stress_slowpath.py iters D t_n mask S dtype
(mask: none | causal | padding)"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_01960_b200 as ta  # noqa: E402

iters, D, t_n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
mask, S = sys.argv[4], int(sys.argv[5])
dt = torch.float16 if sys.argv[6] == "f16" else torch.bfloat16
torch.manual_seed(D * 1000 + S)
B, H = 2, 3
bad = 0
worst = 0.0
for it in range(iters):
    q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=dt) for _ in range(3))
    vl = [S, S // 2 + 7] if mask == "padding" else None
    o = ta.sdpa(q, k, v, scale=1.0, causal=mask == "causal", valid_len=vl,
                schedule=ta.TileSchedule(64, t_n, 2))
    s = torch.einsum("bhqd,bhkd->bhqk", q.float(), k.float())
    if mask == "causal":
        s = s.masked_fill(torch.ones(S, S, device="cuda", dtype=torch.bool).triu(1), -math.inf)
    if vl is not None:
        for b, n in enumerate(vl):
            s[b, :, :, n:] = -math.inf
    ref = torch.softmax(s, -1) @ v.float()
    err = (o.float() - ref).abs().max().item()
    worst = max(worst, err)
    if err > (3e-2 if dt == torch.bfloat16 else 5e-3):
        bad += 1
        print(f"iter {it}: max err {err:.3e}", flush=True)
print(f"D={D} t_n={t_n} mask={mask} S={S} {sys.argv[6]}: {bad} / {iters} bad, worst {worst:.2e}")
