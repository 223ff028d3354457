"""A/B timing of library builds (e.g. -D tuning macros, see _build.py) on one
config (tuning aid).  usage: python scripts/ab_libs.py B H S D lib1 lib2 ..."""
import os, subprocess, sys
B, H, S, D = sys.argv[1:5]
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2603_01960_b200 as ta
B, H, S, D = (int(x) for x in sys.argv[1:5])
q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for _ in range(3): ta.sdpa(q, k, v, out=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n): ta.sdpa(q, k, v, out=o)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
ref = torch.nn.functional.scaled_dot_product_attention(q[:, :2], k[:, :2], v[:, :2])
err = (o[:, :2].float() - ref.float()).abs().max().item()
print(f"{ms:.3f} ms {4*B*H*S*S*D/ms/1e9:7.1f} TF/s err {err:.1e}")
'''
for spec in sys.argv[5:]:
    lib = spec
    env = dict(os.environ, TILEATTN_B200_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", code, B, H, S, D], env=env, capture_output=True, text=True)
    print(f"{os.path.basename(lib):24s}: {(r.stdout.strip() or r.stderr.strip()[-300:])}", flush=True)
