"""Prints per-kernel duration, occupancy, issue and the top warp-stall
reasons of an ncu report (raw page)."""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
col = {n: i for i, n in enumerate(h)}
stall = [n for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    def g(n):
        return r[col[n]] if n in col else "?"
    print("== %s  %s us  regs %s  warps/SM %s  issue%% %s  dram%% %s  L1hit %s" % (
        g("Kernel Name"), g("gpu__time_duration.sum"), g("launch__registers_per_thread"),
        g("sm__warps_active.avg.per_cycle_active"), g("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), g("l1tex__t_sector_hit_rate.pct")))
    vals = []
    for n in stall:
        try:
            vals.append((float(r[col[n]].replace(",", "")), n))
        except ValueError:
            pass
    vals.sort(reverse=True)
    for v, n in vals[:7]:
        print("     %-90s %s" % (n, v))
