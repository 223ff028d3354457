"""Same-box calibration: our kernel (one or more library builds) vs torch SDPA
(cuDNN / flash backend) on a few configs, with the SM clock and power drawn
during each timed region (tuning aid; not the contract bench).

usage: python scripts/calib.py [--torch] [--cfg B,H,S,D[,f16]] ... [lib.so ...]
"""
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CODE = r'''
import sys, json, statistics, torch
sys.path.insert(0, ".")
from bench import ClockSampler
import paper_2603_01960_b200 as ta
cfgs = json.loads(sys.argv[1]); with_torch = sys.argv[2] == "1"
for (B, H, S, D, f16) in cfgs:
    dt = torch.float16 if f16 else torch.bfloat16
    q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=dt) for _ in range(3))
    o = torch.empty_like(q)
    fl = 4 * B * H * S * S * D
    def timed(fn):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        n = max(3, int(1500.0 / max(e0.elapsed_time(e1), 1e-3)))
        for _ in range(n): fn()
        with ClockSampler(torch.cuda.current_device()) as clk:
            e0.record()
            for _ in range(n): fn()
            e1.record(); torch.cuda.synchronize()
        pw = []
        for ln in clk.lines:
            try: pw.append(float(ln.split(",")[3]))
            except Exception: pass
        return e0.elapsed_time(e1) / n, clk.summary()["sm_mhz"], (statistics.median(pw) if pw else None)
    ms, mhz, w = timed(lambda: ta.sdpa(q, k, v, out=o))
    ref = torch.nn.functional.scaled_dot_product_attention(q[:1, :2], k[:1, :2], v[:1, :2])
    err = (o[:1, :2].float() - ref.float()).abs().max().item()
    line = f"B{B} H{H} S{S} D{D} {'f16' if f16 else 'bf16'}: {fl/ms/1e9:7.1f} TF/s ({ms:.3f} ms, {mhz} MHz, {w} W) err {err:.1e}"
    if with_torch:
        ms2, mhz2, w2 = timed(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
        line += f" | torch {fl/ms2/1e9:7.1f} TF/s ({mhz2} MHz, {w2} W)"
    print(line, flush=True)
    del q, k, v, o; torch.cuda.empty_cache()
'''


def main():
    import json
    args = sys.argv[1:]
    cfgs, libs, with_torch = [], [], "0"
    i = 0
    while i < len(args):
        a = args[i]
        if a == "--torch":
            with_torch = "1"
        elif a == "--cfg":
            p = args[i + 1].split(",")
            cfgs.append([int(x) for x in p[:4]] + [len(p) > 4 and p[4] == "f16"])
            i += 1
        else:
            libs.append(a)
        i += 1
    if not cfgs:
        cfgs = [[8, 64, 32768, 128, False]]
    if not libs:
        libs = [str(ROOT / "paper_2603_01960_b200" / "_lib" / "libtileattn_b200.so")]
    for lib in libs:
        env = dict(os.environ, TILEATTN_B200_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", CODE, json.dumps(cfgs), with_torch], env=env,
                           capture_output=True, text=True, cwd=ROOT)
        print(f"== {os.path.basename(lib)}", flush=True)
        print(r.stdout.strip() or r.stderr.strip()[-1500:], flush=True)
        with_torch = "0"  # vendor numbers once per call


if __name__ == "__main__":
    main()
