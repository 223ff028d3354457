"""Same-box A/B timing of library builds over a few configs (tuning aid).

usage: python scripts/ab.py [--tn 64] [--reps 2] CFG... -- lib1.so lib2.so ...
  CFG = B,H,S,D[,f16][,causal]   e.g. 8,64,32768,128  4,16,1024,64,f16
Libraries are interleaved per repetition (power-capped clocks drift between
runs); each line: TF/s, SM clock sampled during the run, max-abs vs torch SDPA
on two heads.
"""
import os
import subprocess
import sys

CODE = r'''
import sys, subprocess, threading, statistics, torch
sys.path.insert(0, ".")
import paper_2603_01960_b200 as ta
B, H, S, D = (int(x) for x in sys.argv[1:5]); flags = sys.argv[5].split(","); tn = int(sys.argv[6])
dt = torch.float16 if "f16" in flags else torch.bfloat16
causal = "causal" in flags
q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=dt) for _ in range(3))
o = torch.empty_like(q)
sched = ta.TileSchedule(64, tn, 2)
st = ta.KernelStats()
import os
if os.environ.get("TILEATTN_B200_LIB", "").endswith("torch"):  # vendor kernel (cuDNN / flash)
    f = lambda: o.copy_(torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)) if False else torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)
    st.block_n = 0
else:
    f = lambda: ta.sdpa(q, k, v, out=o, causal=causal, schedule=sched, stats=st)
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); f(); e1.record(); torch.cuda.synchronize()
n = max(5, int(1500 / max(e0.elapsed_time(e1), 1e-3)))
clk = []
pw = []
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
def _rd():
    for l in p.stdout:
        try:
            a, b = l.split(",")
            clk.append(float(a)); pw.append(float(b))
        except ValueError:
            pass
threading.Thread(target=_rd, daemon=True).start()
e0.record()
for _ in range(n): f()
e1.record(); torch.cuda.synchronize()
p.terminate()
ms = e0.elapsed_time(e1) / n
ref = torch.nn.functional.scaled_dot_product_attention(q[:1, :2], k[:1, :2], v[:1, :2], is_causal=causal)
err = (o[:1, :2].float() - ref.float()).abs().max().item() if st.block_n else 0.0
mhz = statistics.median(clk[len(clk)//3:]) if clk else 0
watt = statistics.median(pw[len(pw)//3:]) if pw else 0
tf = 4*B*H*S*S*D/ms/1e9
print(f"{ms:9.3f} ms {tf:7.1f} TF/s {mhz:5.0f} MHz {watt:5.0f} W {tf/max(mhz,1)*1000:6.1f} TF/s/GHz {tf/max(watt,1):5.2f} TF/J bn={st.block_n} err {err:.1e}")
'''


def main():
    args = sys.argv[1:]
    tn, reps = 128, 2
    while args and args[0].startswith("--"):
        if args[0] == "--tn":
            tn = int(args[1]); args = args[2:]
        elif args[0] == "--reps":
            reps = int(args[1]); args = args[2:]
        else:
            break
    cut = args.index("--")
    cfgs, libs = args[:cut], args[cut + 1:]
    for cfg in cfgs:
        parts = cfg.split(",")
        B, H, S, D = parts[:4]
        flags = ",".join(parts[4:]) or "bf16"
        print(f"== {cfg} (t_n {tn})", flush=True)
        for rep in range(reps):
            for lib in libs:
                env = dict(os.environ, TILEATTN_B200_LIB=os.path.abspath(lib))
                r = subprocess.run([sys.executable, "-c", CODE, B, H, S, D, flags, str(tn)],
                                   env=env, capture_output=True, text=True, timeout=600)
                out = r.stdout.strip() or r.stderr.strip()[-400:]
                print(f"  {os.path.basename(lib):20s} {out}", flush=True)


if __name__ == "__main__":
    main()
