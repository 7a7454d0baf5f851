"""Summarises an ncu --set full report of scripts/profile_configs.py into
profiles/<tag>_ncu_full.md and profiles/ncu_traffic.json (per-launch DRAM
bytes per config/kernel, which bench.py reports as roofline.traffic).

    python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep gpurun_out/ncu_full.log r01
"""
import ast
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, log, tag = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
M = {
    "kernel": "Kernel Name", "us": "gpu__time_duration.sum", "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum", "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread", "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size", "block": "launch__block_size", "smem_dyn": "launch__shared_mem_per_block_dynamic",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
}
col = {k: (h.index(v) if v in h else -1) for k, v in M.items()}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
         "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}


def val(r, k):
    i = col[k]
    if i < 0:
        return None
    v = r[i].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return v.strip()
    return x * scale.get(units[i].strip(), 1)


# launch order -> config (profile_configs.py prints "<config> <tag> [kernels]")
order = []
for line in open(log):
    parts = line.strip().split(" ", 2)
    if len(parts) == 3 and parts[1] in ("fused", "unfused") and parts[2].startswith("["):
        for k in ast.literal_eval(parts[2]):
            order.append((parts[0], parts[1], k))
recs = []
oi = 0
for r in data:
    name = val(r, "kernel")
    while oi < len(order) and order[oi][2] != name:
        oi += 1
    cfg = order[oi][0] if oi < len(order) else "?"
    oi += 1
    recs.append({"config": cfg, **{k: val(r, k) for k in M}})
traffic = {}
lines = ["# ncu --set full summary (%s)" % tag, "",
         "Command: `ncu --set full --clock-control none --import-source on -k regex:'fusion|dbias' "
         "python scripts/profile_configs.py --iters 1` on one B200 (cold L2 per launch, serialised).",
         "DRAM write bytes undercount outputs still dirty in the 126 MB L2 when the kernel ends.", "",
         "| config | kernel | us | DRAM rd MB | DRAM wr MB | DRAM % peak | regs | warps active % | grid x block "
         "| smem B | SM % | FMA % | tensor % | L2 hit % |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]


def f(x, k, d=1):
    return ("%.*f" % (d, x[k])) if isinstance(x[k], float) else str(x[k])


for x in recs:
    lines.append("| %s | %s | %s | %.1f | %.1f | %s | %s | %s | %s x %s | %s | %s | %s | %s | %s |" % (
        x["config"], x["kernel"], f(x, "us"), (x["dram_rd"] or 0) / 1e6, (x["dram_wr"] or 0) / 1e6,
        f(x, "dram_pct"), f(x, "regs", 0), f(x, "warps_active_pct"), f(x, "grid", 0), f(x, "block", 0),
        f(x, "smem_dyn", 0), f(x, "sm_pct"), f(x, "fma_pct"), f(x, "tensor_pct"), f(x, "l2_hit")))
    traffic.setdefault(x["config"], {})[x["kernel"]] = int((x["dram_rd"] or 0) + (x["dram_wr"] or 0))
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "%s_ncu_full.md" % tag), "w") as fh:
    fh.write("\n".join(lines) + "\n")
with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)
print("\n".join(lines))
