"""Small launches of every kernel instantiation for compute-sanitizer.

Run under each tool (one process per tool; ``scripts/sanitize.sh`` does this):
    compute-sanitizer --tool memcheck  python scripts/sanitize.py
    compute-sanitizer --tool synccheck python scripts/sanitize.py
    compute-sanitizer --tool racecheck python scripts/sanitize.py
    compute-sanitizer --tool initcheck python scripts/sanitize.py

Cases: D in {64, 128, 192, 256} (the four instantiations; D=160 runs on the
192-column kernel with the skipped K-steps) x {fp16, bf16} x {none, causal,
padding}, at BASELINE cfg1's shape (B1 H8 S512) and a ragged S (130 / 300),
plus the lazy-rescale slow path (scale 1).  Each result is checked against a
torch fp32 reference so a sanitizer run that silently broke the kernel fails.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_01960_b200 as ta  # noqa: E402


def ref(q, k, v, causal, valid_len, scale):
    qf, kf, vf = q.float(), k.float(), v.float()
    s = torch.einsum("bhqd,bhkd->bhqk", qf, kf) * scale
    S = q.shape[2]
    if causal:
        s = s.masked_fill(torch.ones(S, S, device=q.device, dtype=torch.bool).triu(1), -math.inf)
    if valid_len is not None:
        kk = torch.arange(S, device=q.device)
        for b, n in enumerate(valid_len):
            s[b, :, :, kk >= n] = -math.inf
    lse = torch.logsumexp(s, -1)
    p = torch.softmax(s, -1).nan_to_num(0.0)
    return p @ vf, lse


def main() -> int:
    quick = "--quick" in sys.argv  # one ragged shape per mask and dtype
    only = [a for a in sys.argv[1:] if not a.startswith("--")]  # optional head dims
    torch.manual_seed(0)
    dev = torch.device("cuda:0")
    fails = 0
    n = 0
    dims = [int(x) for x in only] if only else [64, 128, 160, 192, 256]
    for D in dims:
        for dt in (torch.float16, torch.bfloat16):
            for S, B in ((130, 2),) if quick else ((512, 1), (130, 2), (300, 2)):
                for mask in ("none", "causal", "padding"):
                    if S == 512 and dt == torch.bfloat16 and mask != "none":
                        continue
                    H = 8 if S == 512 else 2
                    q, k, v = (torch.randn(B, H, S, D, device=dev, dtype=dt) for _ in range(3))
                    vl = [S - 7, max(0, S // 3)][:B] if mask == "padding" else None
                    scale = 1.0 if (S == 300 and mask == "none") or (quick and mask == "none") \
                        else 1.0 / math.sqrt(D)
                    ro, rl = ref(q, k, v, mask == "causal", vl, scale)
                    # D=128 also on its 64-key kernel (TileSchedule t_n <= 64)
                    for sched in ((None, ta.TileSchedule(64, 64, 2)) if D == 128 else (None,)):
                      o, lse = ta.sdpa(q, k, v, causal=mask == "causal", scale=scale,
                                       return_lse=True, valid_len=vl, schedule=sched)
                      torch.cuda.synchronize()
                      eo = (o.float() - ro).abs().max().item()
                      fin = torch.isfinite(rl)
                      el = (lse[fin] - rl[fin]).abs().max().item() if fin.any() else 0.0
                      # BASELINE tolerance (unit-variance inputs, default scale);
                      # the scale-1 stress case has 8-16x larger scores, so a
                      # peaked softmax whose bf16-rounded P (2^-8 spacing
                      # below 1) moves O by ~|v| 2^-8: 3e-2 there
                      tol = (2e-2 if scale != 1.0 else 3e-2) if dt == torch.bfloat16 else 5e-3
                      ok = eo <= tol and el <= 2e-3 and bool((lse[~fin] == -math.inf).all())
                      n += 1
                      fails += not ok
                      bn = 64 if sched is not None else 128
                      print(f"D={D} {str(dt)[6:]} S={S} B={B} mask={mask} scale={scale:.4g} "
                            f"bn={bn}: max|dO|={eo:.2e} max|dLSE|={el:.2e} "
                            f"{'ok' if ok else 'FAIL'}", flush=True)
    print(f"sanitize cases: {n}, parity failures: {fails}")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
