"""Summarises gpurun_out/launches.csv (ncu gpu__time_duration launch list of
scripts/profile_configs.py --unfused --iters 2) into profiles/<tag>_ncu_launches.md."""
import ast
import csv
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
data = rows[hi + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
order = []
for line in open("gpurun_out/launches.log"):
    p = line.strip().split(" ", 2)
    if len(p) == 3 and p[1] in ("fused", "unfused"):
        order.append((p[0], p[1], ast.literal_eval(p[2])))
out = ["# ncu launch list (%s): gpu__time_duration per launch, --clock-control none" % tag, "",
       "Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/profile_configs.py --unfused --iters 2`",
       "(fused = the bench plan; unfused = one kernel per op). Cold-cache and serialised: compare shares, not absolutes.",
       "Second iteration of each executor; for graphs with >40 kernels only the sum and the 8 largest launches.", "",
       "| config | plan | kernels | sum us | per-kernel us |", "|---|---|---|---|---|"]
seq = [(r[ki].split("(")[0].strip(), float(r[vi]) / 1000) for r in data if not r[ki].startswith("void at::")]
pos = 0
for cfg, kind, ks in order:
    runs = []
    for _ in range(2):
        runs.append(seq[pos:pos + len(ks)])
        pos += len(ks)
    r = runs[1]
    assert [a for a, _ in r] == ks, (cfg, kind)
    shown = r if len(r) <= 40 else sorted(r, key=lambda x: -x[1])[:8]
    out.append("| %s | %s | %d | %.1f | %s |" % (cfg, kind, len(ks), sum(t for _, t in r),
                                               ", ".join("%s %.1f" % (a, t) for a, t in shown)))
open("profiles/%s_ncu_launches.md" % tag, "w").write("\n".join(out) + "\n")
print("\n".join(out[6:]))
