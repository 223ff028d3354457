#!/usr/bin/env python
"""Benchmark of the SDPA forward hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[4], the config the metric's 1/2/4/8-GPU
scaling is quoted on and the largest that fits one GPU):
    long-context B=8 H=64 S=32768 D=128 bf16, non-causal, default scale.
A "step" is one forward over the whole tensor.  At N GPUs each rank owns H/N
heads for every batch (head sharding) — no collective on the
data path; total work is fixed, so scaling is "strong".

Metric: TFLOP/s = 4*B*H*S^2*D / t (reference analysis.cpp:25-30), t the max
over ranks of the CUDA-event time of the K timed steps.  Inputs (2.1 GB) are
far larger than L2 (126 MB), so no flush is needed between steps.

`--impl reference` times the reference's own CPU implementation
(tileattn::sdpa_tiled compiled from its sources into oracle/_ref) on the
host cores: each step is a bounded sample of the same workload — one full
(b,h) head, S=32768, D=128 (1/512 of the job).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOAD = dict(workload="long-context B8 H64 S32K D128 bf16 non-causal (BASELINE configs[4])",
                B=8, H=64, S=32768, D=128, dtype="bf16", causal=False)
METRIC = "SDPA fwd TFLOP/s (4*B*H*S^2*D), B200 vs CPU"
UNIT = "TFLOP/s"


def flops(B, H, S, D):
    return 4.0 * B * H * S * S * D


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(n)
        under_load = [x for x in sm if mx and x > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(under_load) if under_load else None,
                "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline
def cpu_reference_rate(S=32768, D=128, schedules=((64, 128, 2, 0), (128, 128, 2, 1)),
                       runs=1):
    """Reference tileattn::sdpa_tiled (oracle/_ref) on one (b,h) head of the
    workload, all host threads.  Returns (TFLOP/s of the faster schedule, info)."""
    import oracle
    R = oracle.ref("auto")
    q, k, v = oracle.make_input((1, 1, S, D), oracle.BF16, 0)
    h = R.ref_handle_new(q.ravel().copy(), k.ravel().copy(), v.ravel().copy(), 1, 1, S, D,
                         oracle.BF16)
    best = None
    try:
        for (tm, tn, st, lay) in schedules:
            ts = []
            for _ in range(runs):
                t0 = time.perf_counter()
                rc = R.ref_handle_run(h, tm, tn, st, lay, 0, None)
                ts.append(time.perf_counter() - t0)
                if rc != 0:
                    raise RuntimeError(R.ref_last_error())
            t = min(ts)
            if best is None or t < best[0]:
                best = (t, (tm, tn, st, "col" if lay else "row"))
    finally:
        R.ref_handle_free(h)
    rate = flops(1, 1, S, D) / best[0] / 1e12
    return rate, dict(seconds=best[0], schedule=list(best[1]),
                      lib=oracle.ref_variant("auto").name)


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0  # N>1: rank 0 alone runs the CPU reference
    import oracle
    S, D = WORKLOAD["S"], WORKLOAD["D"]
    R = oracle.ref("auto")
    q, k, v = oracle.make_input((1, 1, S, D), oracle.BF16, 0)
    h = R.ref_handle_new(q.ravel().copy(), k.ravel().copy(), v.ravel().copy(), 1, 1, S, D,
                         oracle.BF16)
    sched = (64, 128, 2, 0)  # reference default TileSchedule{} (tiled.hpp:30-37)
    if args.ref_schedule == "col":
        sched = (128, 128, 2, 1)
    try:
        for _ in range(args.warmup):
            R.ref_handle_run(h, *sched, 0, None)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if R.ref_handle_run(h, *sched, 0, None) != 0:
                raise RuntimeError(R.ref_last_error())
        dt = time.perf_counter() - t0
    finally:
        R.ref_handle_free(h)
    ms = dt / args.steps * 1e3
    val = flops(1, 1, S, D) / (dt / args.steps) / 1e12
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) snapped to the bf16 grid (reference make_input, seed 0)",
        "config": dict(WORKLOAD, parallelism="cpu threads"),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"one (b,h) head of the workload per step (S={S}, D={D}; "
                                   f"1/512 of the job), schedule t_m={sched[0]} t_n={sched[1]} "
                                   f"stages={sched[2]} {'col' if sched[3] else 'row'}, "
                                   f"{oracle.ref_variant('auto').name}"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2603_01960_b200 as ta

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2603_01960_b200.sharding import head_range, max_over_ranks
    B, H, S, D = WORKLOAD["B"], WORKLOAD["H"], WORKLOAD["S"], WORKLOAD["D"]
    h0, h1 = head_range(H, world, rank)  # head sharding: this rank owns heads [h0, h1)
    Hl = h1 - h0
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    q, k, v = (torch.randn(B, Hl, S, D, device=dev, generator=g, dtype=torch.bfloat16)
               for _ in range(3))
    o = torch.empty_like(q)
    stream = torch.cuda.current_stream(dev)
    stats = ta.KernelStats()

    def step():
        ta.sdpa(q, k, v, out=o, stats=stats)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---- device-timed region: K steps, one event pair per step on the
    # launching stream (kernel launch duration = step duration here)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for e0, e1 in evs:
            e0.record(stream)
            step()
            e1.record(stream)
        t_end.record(stream)
        barrier()
    total_ms = t_start.elapsed_time(t_end)
    per_launch = [e0.elapsed_time(e1) for e0, e1 in evs]
    if world > 1:
        total_ms = max_over_ranks(total_ms, device=dev)
    ms_step = total_ms / args.steps
    job_flops = flops(B, H, S, D)
    value = job_flops / (ms_step / 1e3) / 1e12

    # ---- roofline of the dominant (only) kernel, per launch
    pk, pk_kind = peaks()
    launch_ms = statistics.mean(per_launch)
    achieved = flops(B, Hl, S, D) / (launch_ms / 1e3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            ps = json.loads(prof.read_text())
            if ps.get("workload") == WORKLOAD["workload"] and world == 1:
                traffic = ps.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops"], "traffic": traffic,
                "peak_kind": f"{pk_kind} burst bf16 (MEASURED_PEAKS.json bf16_tflops)",
                "frac_of_sustained": achieved / pk.get("bf16_tflops_sustained",
                                                       pk["bf16_tflops"]),
                "algorithmic_bytes_per_launch": 8 * B * Hl * S * D + 4 * B * Hl * S}

    # ---- e2e through the public host-buffer entry (ta_sdpa_fwd_host):
    # pinned host q/k/v -> H2D, kernel, D2H of O, every step
    e2e = None
    if not args.no_e2e:
        hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
        ho = torch.empty_like(hq).pin_memory()
        shape = (B, Hl, S, D)
        ptrs = (hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), ho.data_ptr())

        def e2e_step():
            ta.sdpa_fwd_host(*ptrs, 0, shape, ta.BF16, stream=stream.cuda_stream)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        n_e2e = max(1, min(args.steps, 5))
        for _ in range(n_e2e):
            e2e_step()
        barrier()
        e2e_s = (time.perf_counter() - t0) / n_e2e
        if world > 1:
            e2e_s = max_over_ranks(e2e_s, device=dev)
        nbytes = q.numel() * 2
        e2e = {"value": job_flops / e2e_s / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": 3 * nbytes * world, "d2h_bytes_per_step": nbytes * world,
               "ms_per_step": e2e_s * 1e3, "steps": n_e2e,
               "path": "ta_sdpa_fwd_host (C-ABI, pinned host buffers, includes copies)"}
        del hq, hk, hv, ho

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rate, info = cpu_reference_rate()
            cpu = {"value": rate, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"one (b,h) head of the workload (S=32768, D=128; 1/512 of the "
                             f"job), best of schedules {{64,128,2,row}}/{{128,128,2,col}} -> "
                             f"{info['schedule']}, {info['seconds']:.2f} s, {info['lib']}"}
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic N(0,1) bf16 (torch.randn on device, seed 1234+rank)",
            "config": dict(WORKLOAD, parallelism=f"head-shard{world}", heads_per_gpu=Hl,
                           l2="inputs 2.1 GB >> 126 MB L2; no flush needed"),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": args.steps,
            "kernel": {"name": "ta::sdpa_fwd_kernel<128,bf16>", "ctas": stats.ctas,
                       "block_m": stats.block_m, "block_n": stats.block_n,
                       "stages": stats.stages, "q_tiles_per_cta": stats.q_tiles_per_cta,
                       "per_launch_ms": [round(x, 4) for x in per_launch]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_sweep(args):
    """All BASELINE configs on one GPU (report table; not the contract line)."""
    import torch
    import paper_2603_01960_b200 as ta
    pk, _ = peaks()
    configs = [
        ("cfg1 B1 H8 S512 D64 f16", 1, 8, 512, 64, torch.float16),
        *[(f"S-sweep B4 H16 S{s} D64 bf16", 4, 16, s, 64, torch.bfloat16)
          for s in (1024, 2048, 4096, 8192, 16384)],
        *[(f"D-sweep B8 H32 S4096 D{d} {n}", 8, 32, 4096, d, t) for d in (64, 96, 128, 160, 256)
          for n, t in (("f16", torch.float16), ("bf16", torch.bfloat16))],
        ("ViT B64 H16 S1024 D64 bf16", 64, 16, 1024, 64, torch.bfloat16),
        ("long B8 H64 S32768 D128 bf16", 8, 64, 32768, 128, torch.bfloat16),
    ]
    # causal twins (half the paper's grid): same FLOP convention
    # as the reference's flop_rate (4*B*H*S^2*D); "causal_effective_tflops"
    # counts the admitted half only
    causal = [("D-sweep B8 H32 S4096 D128 bf16 causal", 8, 32, 4096, 128, torch.bfloat16),
              ("long B8 H64 S32768 D128 bf16 causal", 8, 64, 32768, 128, torch.bfloat16)]
    rows = []
    for name, B, H, S, D, dt in configs + causal:
        is_causal = name.endswith("causal")
        q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=dt) for _ in range(3))
        o = torch.empty_like(q)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def timed(fn):
            # warm up for >= 0.2 s (clocks settle under the power cap after
            # the previous config), then time >= 0.2 s of back-to-back calls
            fn()
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            n = max(3, int(200.0 / max(e0.elapsed_time(e1), 1e-3)))
            for _ in range(n):
                fn()
            e0.record()
            for _ in range(n):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n

        ms = timed(lambda: ta.sdpa(q, k, v, out=o, causal=is_causal))
        tf = flops(B, H, S, D) / ms / 1e9
        ref_ms = None
        if args.vendor:
            ref_ms = timed(lambda: torch.nn.functional.scaled_dot_product_attention(
                q, k, v, is_causal=is_causal))
        rows.append(dict(config=name, ms=ms, tflops=tf, frac=tf / pk["bf16_tflops"],
                         causal_effective_tflops=tf / 2 if is_causal else None,
                         hbm_gbs=(8 * B * H * S * D + 4 * B * H * S) / ms / 1e6,
                         torch_sdpa_ms=ref_ms,
                         torch_sdpa_tflops=(flops(B, H, S, D) / ref_ms / 1e9) if ref_ms else None))
        print(json.dumps(rows[-1]), flush=True)
        del q, k, v, o
        torch.cuda.empty_cache()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-schedule", choices=["row", "col"], default="row")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="all BASELINE configs (report only)")
    ap.add_argument("--vendor", action="store_true", help="with --sweep: time torch SDPA too")
    args = ap.parse_args()
    if args.warmup < 3 and not args.sweep and args.impl == "ours":
        print("note: warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.sweep:
        return run_sweep(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
