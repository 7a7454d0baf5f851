"""Per-launch table of an ncu launch-list capture of scripts/profile_configs.py
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
lts__t_sectors_srcunit_tex_op_write.sum --csv): one row per stitched kernel
with its duration, DRAM reads, DRAM writes and the bytes its stores wrote
into L2 (lts write sectors x 32). Writes that are still dirty in the 126 MB L2
when a kernel ends are not in dram__bytes_write (the write-back happens
later), so the traffic a kernel causes is counted as

    traffic = dram__bytes_read + max(dram__bytes_write, lts write bytes)

-- the stores it issued all reach DRAM eventually. Also writes
profiles/ncu_traffic.json ({config: {kernel: traffic bytes per launch}}),
which bench.py reports as roofline.traffic.

    python scripts/ncu_launch_table.py gpurun_out/launches.csv gpurun_out/launches.log r02
"""
import ast
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, log, tag = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
launches = {}
order = []
for r in rows[hi + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    i = int(d["ID"])
    if i not in launches:
        launches[i] = {"name": d["Kernel Name"].split("(")[0]}
        order.append(i)
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
             "sector": 32}.get(unit, 1)
    launches[i][d["Metric Name"]] = v * scale
# stitched kernels only (torch's randn / empty kernels are skipped)
ours = [launches[i] for i in order if not launches[i]["name"].startswith(("void ", "at::"))]
seqs = []
for line in open(log):
    parts = line.split(" ", 2)
    if len(parts) == 3 and parts[2].startswith("["):
        seqs.append((parts[0], parts[1], ast.literal_eval(parts[2].strip())))
out_md = ["# ncu launch list (%s): per-launch time and DRAM / L2-write traffic" % tag, "",
          "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
          "lts__t_sectors_srcunit_tex_op_write.sum --clock-control none` of `scripts/profile_configs.py --iters 1` "
          "(serialised launches, cold L2 between configs; a profiler time is never a bench value). "
          "traffic = DRAM read + max(DRAM write, L2 write bytes).", ""]
traffic = {}
pos = 0
for cfg, kind, seq in seqs:
    out_md += ["## %s (%s, %d launches)" % (cfg, kind, len(seq)), "",
               "| kernel | us | DRAM read MB | DRAM write MB | L2 write MB | traffic MB |", "|---|---|---|---|---|---|"]
    tot = [0.0] * 5
    # the dataflow launch issues in its own (topological) order: match this
    # config's launches by name, list them in schedule order
    chunk = ours[pos:pos + len(seq)]
    pos += len(seq)
    assert sorted(x["name"] for x in chunk) == sorted(seq), (cfg, kind)
    by_name = {x["name"]: x for x in chunk}
    for name in seq:
        L = by_name[name]
        us = L.get("gpu__time_duration.sum", 0)
        rd = L.get("dram__bytes_read.sum", 0)
        wr = L.get("dram__bytes_write.sum", 0)
        l2w = L.get("lts__t_sectors_srcunit_tex_op_write.sum", 0)
        t = rd + max(wr, l2w)
        traffic.setdefault(cfg, {})[name] = t
        for j, x in enumerate((us, rd, wr, l2w, t)):
            tot[j] += x
        out_md.append("| %s | %.2f | %.1f | %.1f | %.1f | %.1f |" % (name, us, rd / 1e6, wr / 1e6, l2w / 1e6, t / 1e6))
    out_md.append("| **total** | %.1f | %.1f | %.1f | %.1f | %.1f |" % (tot[0], tot[1] / 1e6, tot[2] / 1e6, tot[3] / 1e6,
                                                                       tot[4] / 1e6))
    out_md.append("")
with open(os.path.join(ROOT, "profiles", "%s_ncu_launches.md" % tag), "w") as f:
    f.write("\n".join(out_md) + "\n")
with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1, sort_keys=True)
print("kernels:", pos, "configs:", [s[0] for s in seqs])
