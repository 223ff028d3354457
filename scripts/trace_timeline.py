"""Cycle timeline of CTA (0,0) for one config (diagnostics).
usage: python scripts/trace_timeline.py B H S D"""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2603_01960_b200 as ta

B, H, S, D = (int(x) for x in sys.argv[1:5])
q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for _ in range(3):
    ta.sdpa(q, k, v, out=o)
tr = torch.zeros(24 * 64, dtype=torch.int64, device="cuda")
L = ta.lib()
L.ta_debug_sdpa_trace.restype = ctypes.c_int
L.ta_debug_sdpa_trace.argtypes = [ctypes.c_void_p] * 4 + [ta._Shape, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
ta._check(L.ta_debug_sdpa_trace(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), ta._Shape(B, H, S, D), ta.BF16, tr.data_ptr(), None))
t = tr.view(24, 64).cpu().numpy()
names = ["mmaWaitP0", "mmaIssPV0", "mmaWaitP1", "mmaIssPV1", "s0Ready", "s0Load", "s0Max", "s0Exp", "s0Arrive", "s1Ready", "s1Load", "s1Max", "s1Exp", "s1Arrive", "tcPV0", "tcS0", "tcPV1", "tcS1"]
base = t[4, 0]
n = min(64, (S + 127) // 128)
print("iter " + " ".join(f"{x:>9s}" for x in names))
for j in range(n):
    print(f"{j:4d} " + " ".join(f"{(t[e, j] - base) if t[e, j] else 0:9d}" for e in range(18)))
import numpy as np
print(f"kernel start {t[21, 0] - base}, after setup {t[21, 1] - base}, "
      f"epilogue done tile0 {t[22, 0] - base} tile1 {t[22, 1] - base}, "
      f"last P arrive tile0 {t[8, min(n, 64) - 1] - base} tile1 {t[13, min(n, 64) - 1] - base}")
js = range(8, n - 1)
def d(a, b): return np.mean([t[b, j] - t[a, j] for j in js])
print("mean over iters 8..n-2 (cycles):")
print(" period s0Ready->s0Ready", np.mean([t[4, j + 1] - t[4, j] for j in js]))
print(" s0: ready->load %.0f load->max %.0f max->exp %.0f exp->arrive %.0f" % (d(4, 5), d(5, 6), d(6, 7), d(7, 8)))
print(" s0: arrive(j) -> ready(j+1) %.0f" % np.mean([t[4, j + 1] - t[8, j] for j in js]))
if t[2, 8] and not t[9, 8]:  # one Q tile per CTA (D=64): MMA-warp view of S(j+1)
    print(" QT=1: ready(j) -> mma sees s_read(j) %.0f, -> S(j+1) issued %.0f, -> S(j+1) done %.0f, "
          "mma issued PV(j) -> S(j+1) issued %.0f" % (
              np.mean([t[2, j] - t[4, j] for j in js]), np.mean([t[3, j] - t[4, j] for j in js]),
              np.mean([t[15, j + 1] - t[4, j] for j in js]), np.mean([t[3, j + 1] - t[1, j] for j in js])))
    print(" QT=1: last warp arrive(j) = max(w0..w3) -> mma sees P(j) %.0f" % np.mean(
        [t[0, j] - max(t[8, j], *(t[17 + w, j] for w in (1, 2, 3))) for j in js]))
print(" s1: ready->load %.0f load->max %.0f max->exp %.0f exp->arrive %.0f" % (d(9, 10), d(10, 11), d(11, 12), d(12, 13)))
print(" tile-0 warp skew (warp w arrive - warp 0 arrive) w=1,2,3:", [np.mean([t[17 + w, j] - t[8, j] for j in js]) for w in (1, 2, 3)])
print(" s0 arrive(j) -> mma sees P0(j):", np.mean([t[0, j] - t[8, j] for j in js]))
print(" mma saw P0(j) -> PV0(j) issued:", np.mean([t[1, j] - t[0, j] for j in js]))
print(" s1 arrive(j) -> mma sees P1(j):", np.mean([t[2, j] - t[13, j] for j in js]))
print(" PV0(j) issued -> s0 ready(j+1):", np.mean([t[4, j + 1] - t[1, j] for j in js]))
print(" TC: PV0(j) done -> S0(j+1) done %.0f" % d(14, 15))
print(" TC: S0(j+1) done -> PV1(j) done %.0f" % d(15, 16))
print(" TC: PV1(j) done -> S1(j+1) done %.0f" % d(16, 17))
print(" TC: S1(j+1) done -> PV0(j+1) done %.0f" % np.mean([t[14, j + 1] - t[17, j] for j in js]))
print(" s0 P-half1 arrive(j) -> PV0(j) done %.0f" % np.mean([t[14, j] - t[8, j] for j in js]))
print(" s1 P-half1 arrive(j) -> PV1(j) done %.0f" % np.mean([t[16, j] - t[13, j] for j in js]))
