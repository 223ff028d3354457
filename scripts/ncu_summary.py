"""Summarise an ncu --set full report of the SDPA kernel into profiles/.
usage: python scripts/ncu_summary.py gpurun_out/prof_long.ncu-rep profiles/r01/ncu_long.json [workload]"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "sm__cycles_elapsed.avg": "sm_cycles",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12,
         "ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1.0}
launches = []
for r in rows[2:]:
    d = {}
    for h, u, v in zip(hdr, units, r):
        if h in keys:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            d[keys[h]] = x * scale.get(u, 1.0)
    if "Kernel Name" in hdr:
        d["kernel"] = r[hdr.index("Kernel Name")][:120]
    launches.append(d)
k = launches[0]
summary = {
    "report": rep, "workload": workload, "kernel": k.get("kernel"),
    "duration_s": k.get("duration"),
    "dram_bytes_per_launch": (k.get("dram_read", 0) + k.get("dram_write", 0)) or None,
    "dram_read_bytes": k.get("dram_read"), "dram_write_bytes": k.get("dram_write"),
    **{x: k.get(x) for x in ("tensor_pipe_active_pct", "xu_pipe_pct", "fma_pipe_pct", "alu_pipe_pct",
                             "issue_active_pct", "registers_per_thread", "grid_size", "block_size",
                             "sm_cycles", "l2_hit_rate_pct", "dram_throughput_pct")},
    "note": "ncu --set full --clock-control none (cold caches, replayed): compare shares, not absolute time",
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
