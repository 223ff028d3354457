"""Quick correctness probe of a library build (TILEATTN_B200_LIB) on a few
shapes against torch fp32 (tuning aid; run under `timeout`).
usage: python scripts/probe.py D [D ...]"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_01960_b200 as ta  # noqa: E402


def ref(q, k, v, vl=None, causal=False):
    s = torch.einsum("bhqd,bhkd->bhqk", q.float(), k.float()) / math.sqrt(q.shape[-1])
    S = q.shape[2]
    if causal:
        s = s.masked_fill(torch.ones(S, S, device=q.device, dtype=torch.bool).triu(1), -math.inf)
    if vl is not None:
        for b, n in enumerate(vl):
            s[b, :, :, n:] = -math.inf
    return torch.softmax(s, -1).nan_to_num(0.0) @ v.float(), torch.logsumexp(s, -1)


bad = 0
for D in [int(x) for x in sys.argv[1:]] or [128]:
    for (B, H, S, vl, causal) in [(1, 2, 512, None, False), (2, 3, 300, None, False),
                                  (2, 2, 700, [700, 333], False), (1, 2, 256, None, False),
                                  (1, 1, 129, None, False), (2, 2, 1, None, False),
                                  (1, 4, 4096, None, False), (1, 2, 640, None, True),
                                  (3, 2, 384, [0, 100, 384], False)]:
        for dt in (torch.bfloat16, torch.float16):
            q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=dt) for _ in range(3))
            o, lse = ta.sdpa(q, k, v, return_lse=True, valid_len=vl, causal=causal)
            torch.cuda.synchronize()
            ro, rl = ref(q, k, v, vl, causal)
            eo = (o.float() - ro).abs().max().item()
            fin = torch.isfinite(rl)
            el = (lse[fin] - rl[fin]).abs().max().item() if fin.any() else 0.0
            ok = eo <= (2e-2 if dt == torch.bfloat16 else 5e-3) and el <= 1e-3
            bad += not ok
            print(f"D={D} {str(dt)[6:]} B{B} H{H} S{S} vl={vl} causal={causal}: "
                  f"dO={eo:.2e} dLSE={el:.2e} {'ok' if ok else 'FAIL'}", flush=True)
print("failures:", bad)
sys.exit(1 if bad else 0)
