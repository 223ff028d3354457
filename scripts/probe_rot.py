"""Diagnostics: which (head, row) of a D=64 run disagree with torch SDPA, per
library build.  usage: python scripts/probe_rot.py lib1.so lib2.so ..."""
import os, subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2603_01960_b200 as ta
torch.manual_seed(0)
for (B,H,S) in [(1,1,4096),(1,8,4096),(4,16,4096)]:
    q, k, v = (torch.randn(B, H, S, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = ta.sdpa(q, k, v)
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float())
    bad = ~((o.float() - ref).abs() < 2e-2)
    rows = bad.any(-1).view(-1, S)
    blk = rows.view(-1, 128).any(-1).nonzero().flatten().tolist()
    print(B, H, S, "bad rows", int(rows.sum()), "bad blocks (idx)", len(blk), blk[:12])
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, TILEATTN_B200_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print(f"== {os.path.basename(lib)}\n{(r.stdout.strip() or r.stderr.strip()[-500:])}", flush=True)
