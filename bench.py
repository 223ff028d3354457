#!/usr/bin/env python
"""Benchmark of the SDPA forward hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[4], the config the metric's 1/2/4/8-GPU
scaling is quoted on and the largest that fits one GPU):
    long-context B=8 H=64 S=32768 D=128 bf16, non-causal, default scale.
A "step" is one forward (O and LSE) over the whole tensor.  At N GPUs each
rank owns H/N heads for every batch (head sharding) — no
collective on the data path; total work is fixed, so scaling is "strong".
`--gpus N` under torchrun uses its environment; without a launcher bench.py
starts the N ranks itself (one process per GPU, 127.0.0.1 rendezvous).

Metric: TFLOP/s = 4*B*H*S^2*D / t (reference analysis.cpp:25-30), t the max
over ranks of the CUDA-event time of the K timed steps; per-step median and
nearest-rank p95 as the reference harness reports them (bench.cpp:19-33).
Inputs (3 x 4.3 GB) are far larger than L2 (126 MB), so no flush is needed
between steps.

`--impl reference` times the reference's own CPU implementation
(tileattn::sdpa_tiled compiled from its sources into oracle/_ref) on the
host cores: each step is a bounded sample of the same workload — one full
(b,h) head, S=32768, D=128 (1/512 of the job), the same bytes as the GPU
arm's first head.
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


# ------------------------------------------------------------ inputs
SEED = 1234


def sample_head(S, D, seed=SEED):
    """(q, k, v) of head (b=0, h=0) of rank 0's input, generated on the host
    (torch CPU generator, N(0,1) snapped to bf16): the GPU arm uploads these
    exact bytes as its first head and both CPU arms (cpu_baseline and
    --impl reference) time the reference on them (identical bytes)."""
    import torch
    g = torch.Generator().manual_seed(seed)
    return tuple(torch.randn(S, D, generator=g).to(torch.bfloat16) for _ in range(3))


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def quantiles(samples):
    """Median and nearest-rank p95 exactly as the reference harness
    (bench.cpp:19-33): p95 = sorted[ceil(0.95 n) - 1] in integer arithmetic."""
    xs = sorted(samples)
    n = len(xs)
    med = xs[n // 2] if n % 2 else 0.5 * (xs[n // 2 - 1] + xs[n // 2])
    return med, xs[(19 * n + 19) // 20 - 1]


# ------------------------------------------------------------ CPU baseline
SCHEDULES = {"row": (64, 128, 2, 0),   # reference default TileSchedule{} (tiled.hpp:30-37)
             "col": (128, 128, 2, 1)}  # the reference's faster layout on this path


class _RefHead:
    """The reference tileattn::sdpa_tiled (oracle/_ref) on one (b,h) head."""

    def __init__(self, S, D):
        import numpy as np
        import oracle
        self.S, self.D = S, D
        self.R = oracle.ref("auto")
        self.lib_name = oracle.ref_variant("auto").name
        q, k, v = (np.ascontiguousarray(x.float().numpy()).ravel() for x in sample_head(S, D))
        self.h = self.R.ref_handle_new(q, k, v, 1, 1, S, D, oracle.BF16)

    def run(self, sched):
        if self.R.ref_handle_run(self.h, *sched, 0, None) != 0:
            raise RuntimeError(self.R.ref_last_error())

    def time(self, sched, steps, warmup):
        for _ in range(warmup):
            self.run(sched)
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            self.run(sched)
            ts.append(time.perf_counter() - t0)
        return ts

    def close(self):
        self.R.ref_handle_free(self.h)


def cpu_reference_rate(S=32768, D=128):
    """cpu_baseline leg: both reference schedules on one head of the workload,
    all host threads, one run each.  Returns (TF/s of the faster, info)."""
    ref = _RefHead(S, D)
    try:
        secs = {name: ref.time(sc, 1, 0)[0] for name, sc in SCHEDULES.items()}
    finally:
        ref.close()
    best = min(secs, key=secs.get)
    rates = {n: flops(1, 1, S, D) / t / 1e12 for n, t in secs.items()}
    return rates[best], dict(seconds=secs, rates=rates, best=best, lib=ref.lib_name)


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0  # N>1: rank 0 alone runs the CPU reference
    S, D = args.cpu_sample_s, WORKLOAD["D"]
    ref = _RefHead(S, D)
    try:
        # value: the faster reference schedule (col) over K steps; the
        # default schedule (row) is timed beside it over min(K, 2) steps
        ts = {"col": ref.time(SCHEDULES["col"], args.steps, args.warmup),
              "row": ref.time(SCHEDULES["row"], min(args.steps, 2), min(args.warmup, 1))}
    finally:
        ref.close()
    per = {n: flops(1, 1, S, D) / (sum(t) / len(t)) / 1e12 for n, t in ts.items()}
    ms = sum(ts["col"]) / len(ts["col"]) * 1e3
    val = per["col"]
    cores = os.cpu_count()
    med, p95 = quantiles([t * 1e3 for t in ts["col"]])
    sample = (f"one (b,h) head of the workload per step (S={S}, D={D}; "
              f"{'1/512 of the job' if S == 32768 else 'reduced S'}), bytes identical to the "
              f"GPU arm's head 0; schedule {{128,128,2,col}} (the faster; default "
              f"{{64,128,2,row}} measured {per['row']:.4f} TF/s), {ref.lib_name}")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "ms_per_step_median": med, "ms_per_step_p95": p95,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) snapped to bf16 (torch CPU generator, seed 1234)",
        "config": dict(WORKLOAD, parallelism="cpu threads"),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(),
                         "kind": "reference", "sample": sample,
                         "schedules": {"col": per["col"], "row": per["row"]}},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ launch
def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """`python bench.py --gpus N` with no launcher: start N local ranks (one
    process per GPU, the torchrun environment), rank 0's stdout is the
    output; other ranks' stdout goes to stderr."""
    port = _free_port()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()),
                                       *sys.argv[1:]], env=env,
                                      stdout=None if r == 0 else sys.stderr))
    rcs = [p.wait() for p in procs]
    return max(rcs)


# ------------------------------------------------------------------ our arm
class _EventClock:
    """CUDA events on the launching stream (device time)."""

    def __init__(self, stream):
        import torch
        self.torch, self.stream = torch, stream

    def mark(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def ms(self, a, b):
        return a.elapsed_time(b)


class _HostClock:
    """--stub-step (CPU orchestration test): host wall clock."""

    def mark(self):
        return time.perf_counter()

    def ms(self, a, b):
        return (b - a) * 1e3


def timed_steps(step, clock, steps, warmup, barrier):
    """W untimed steps, then exactly K timed steps bracketed by barrier +
    synchronize on both sides; one mark pair per step.  Returns (total ms of
    the K steps on this rank, per-step ms)."""
    for _ in range(warmup):
        step()
    barrier()
    marks = []
    t_start = clock.mark()
    for _ in range(steps):
        a = clock.mark()
        step()
        marks.append((a, clock.mark()))
    t_end = clock.mark()
    barrier()
    return clock.ms(t_start, t_end), [clock.ms(a, b) for a, b in marks]


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    stub = args.stub_step
    if stub:
        dev = torch.device("cpu")
        if world > 1:
            dist.init_process_group("gloo", rank=rank, world_size=world)
    elif args.share_device:
        # GPU test mode: every rank on cuda:0 (gloo), exercising the
        # multi-rank GPU flow on a one-GPU box; not a scaling measurement
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        if world > 1:
            dist.init_process_group("gloo", rank=rank, world_size=world)
    else:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        if world > 1:
            # NCCL communicator lines (nranks) in the log; nothing on the
            # data path uses it (barriers and the max-over-ranks timing only)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)

    red_dev = torch.device("cpu") if (stub or args.share_device) else dev  # (gloo: host tensors)
    from paper_2603_01960_b200.sharding import head_range, max_over_ranks
    B, H, S, D = WORKLOAD["B"], WORKLOAD["H"], WORKLOAD["S"], WORKLOAD["D"]
    h0, h1 = head_range(H, world, rank)  # head sharding: this rank owns heads [h0, h1)
    Hl = h1 - h0

    def barrier():
        if world > 1:
            dist.barrier()
        if not stub:
            torch.cuda.synchronize(dev)

    stats = None
    if stub:
        # orchestration test only: a fixed CPU step stands in for the kernel
        a = torch.randn(192, 192)
        step = lambda: a @ a  # noqa: E731
        clock = _HostClock()
        job_flops = flops(B, H, S, D)
    else:
        import paper_2603_01960_b200 as ta
        g = torch.Generator(device=dev).manual_seed(SEED + rank)
        q, k, v = (torch.randn(B, Hl, S, D, device=dev, generator=g, dtype=torch.bfloat16)
                   for _ in range(3))
        if rank == 0:  # head 0: the bytes the CPU arms time (sample_head)
            for x, hx in zip((q, k, v), sample_head(S, D)):
                x[0, 0].copy_(hx)
        o = torch.empty_like(q)
        lse = torch.empty((B, Hl, S), device=dev, dtype=torch.float32)
        stream = torch.cuda.current_stream(dev)
        stats = ta.KernelStats()

        def step():
            ta.sdpa(q, k, v, out=o, return_lse=True, lse_out=lse, stats=stats)

        clock = _EventClock(stream)
        job_flops = flops(B, H, S, D)

    sampler = ClockSampler(local) if not stub else None
    if sampler:
        sampler.__enter__()
    try:
        total_ms, per_step = timed_steps(step, clock, args.steps, args.warmup, barrier)
    finally:
        if sampler:
            sampler.__exit__(None, None, None)
    if world > 1:
        total_ms = max_over_ranks(total_ms, device=red_dev)
        per_step = [max_over_ranks(x, device=red_dev) for x in per_step]
    ms_step = total_ms / args.steps
    value = job_flops / (ms_step / 1e3) / 1e12
    med, p95 = quantiles(per_step)

    # ---- roofline of the dominant (only) kernel, per launch
    pk, pk_kind = peaks()
    launch_ms = statistics.mean(per_step)
    achieved = flops(B, Hl, S, D) / (launch_ms / 1e3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists() and not stub:
        try:
            ps = json.loads(prof.read_text())
            if ps.get("workload") == WORKLOAD["workload"] and world == 1:
                traffic = ps.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops"], "traffic": traffic,
                "traffic_source": "profiles/ncu_summary.json (ncu --set full of this workload)",
                "peak_kind": f"{pk_kind} burst bf16 (MEASURED_PEAKS.json bf16_tflops)",
                "frac_of_sustained": achieved / pk.get("bf16_tflops_sustained",
                                                       pk["bf16_tflops"]),
                "algorithmic_bytes_per_launch": 8 * B * Hl * S * D + 4 * B * Hl * S}

    # ---- e2e through the public host-buffer entry (ta_sdpa_fwd_host):
    # pinned host q/k/v -> H2D, kernel, D2H of O and LSE, every step
    e2e = None
    if not args.no_e2e and not stub:
        hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
        ho = torch.empty_like(hq).pin_memory()
        hl = torch.empty((B, Hl, S), dtype=torch.float32).pin_memory()
        shape = (B, Hl, S, D)
        ptrs = (hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), ho.data_ptr(), hl.data_ptr())

        def e2e_step():
            ta.sdpa_fwd_host(*ptrs, shape, ta.BF16, stream=stream.cuda_stream)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        n_e2e = max(1, min(args.steps, 5))
        for _ in range(n_e2e):
            e2e_step()
        barrier()
        e2e_s = (time.perf_counter() - t0) / n_e2e
        if world > 1:
            e2e_s = max_over_ranks(e2e_s, device=red_dev)
        nbytes = B * H * S * D * 2
        e2e = {"value": job_flops / e2e_s / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": 3 * nbytes, "d2h_bytes_per_step": nbytes + 4 * B * H * S,
               "ms_per_step": e2e_s * 1e3, "steps": n_e2e,
               "path": "ta_sdpa_fwd_host (C-ABI, pinned host buffers, includes copies of "
                       "q/k/v in and O/LSE out)"}
        del hq, hk, hv, ho, hl

    # ---- CPU baseline: rank 0, every N (bounded sample, after the timed
    # region; the other ranks wait at the final barrier)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            rate, info = cpu_reference_rate(S=args.cpu_sample_s, D=D)
            cpu = {"value": rate, "unit": UNIT, "cores": os.cpu_count(),
                   "cpu_model": cpu_model(), "kind": "reference",
                   "sample": f"one (b,h) head of the workload (S={args.cpu_sample_s}, D={D}; "
                             f"bytes identical to the GPU arm's head 0), schedules "
                             f"{{64,128,2,row}} {info['rates']['row']:.4f} / "
                             f"{{128,128,2,col}} {info['rates']['col']:.4f} TF/s -> best "
                             f"{info['best']}, {info['lib']}",
                   "schedules": info["rates"]}
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "ms_per_step_median": med, "ms_per_step_p95": p95,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic N(0,1) bf16 (torch.randn on device, seed 1234+rank; head 0 of "
                    "rank 0 = the CPU arms' sample head)",
            "config": dict(WORKLOAD, parallelism=f"head-shard{world}", heads_per_gpu=Hl,
                           l2="inputs 3 x 4.3 GB >> 126 MB L2; no flush needed"),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": sampler.summary() if sampler else None,
            "gpu_launches": 0 if stub else args.steps,
        }
        if stub:
            line["stub"] = "orchestration test: CPU step, gloo, host clock (not a measurement)"
        if args.share_device:
            line["shared_device"] = ("test mode: all ranks on cuda:0 over gloo "
                                     "(not a scaling measurement)")
        if not stub:
            line["kernel"] = {"name": "ta::sdpa_fwd_kernel<128,bf16>", "ctas": stats.ctas,
                              "block_m": stats.block_m, "block_n": stats.block_n,
                              "stages": stats.stages, "q_tiles_per_cta": stats.q_tiles_per_cta,
                              "per_launch_ms": [round(x, 4) for x in per_step]}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:  # last, after NCCL's teardown messages: the output's final line
        print(json.dumps(line), flush=True)
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
    ap.add_argument("--cpu-sample-s", type=int, default=WORKLOAD["S"],
                    help="S of the CPU arms' one-head sample (default: the workload's)")
    ap.add_argument("--stub-step", action="store_true",
                    help="CPU orchestration test (gloo, stub step); not a measurement")
    ap.add_argument("--share-device", action="store_true",
                    help="GPU test mode: all ranks on cuda:0 over gloo; not a measurement")
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.sweep:
        return spawn_ranks(args)
    if args.sweep:
        return run_sweep(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
