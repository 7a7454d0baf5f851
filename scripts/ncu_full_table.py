"""One markdown row per kernel of ncu --set full reports: time, DRAM read /
write, L2-write bytes, traffic, achieved DRAM throughput, SM issue, warps
active, registers, tensor pipe.
    python scripts/ncu_full_table.py out.md rep1.ncu-rep [rep2 ...]"""
import csv
import io
import subprocess
import sys

out, reps = sys.argv[1], sys.argv[2:]
K = [("gpu__time_duration.sum", "us", 1), ("dram__bytes_read.sum", "DRAM rd MB", 1e-6),
     ("dram__bytes_write.sum", "DRAM wr MB", 1e-6), ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 wr MB", 32e-6),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", 1),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
     ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %", 1),
     ("launch__registers_per_thread", "regs", 1), ("launch__block_size", "block", 1), ("launch__grid_size", "grid", 1)]
lines = ["| report | kernel | " + " | ".join(k[1] for k in K) + " |", "|" + "---|" * (len(K) + 2)]
for rep in reps:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        vals = []
        for m, _, sc in K:
            v = d.get(m, "")
            try:
                x = float(v.replace(",", ""))
                u = units[h.index(m)]
                if m.startswith("gpu__time") and u in ("ns", "nsecond"):
                    x *= 1e-3
                if u in ("Mbyte",) and sc == 1e-6:
                    x *= 1e6
                if u in ("Kbyte",) and sc == 1e-6:
                    x *= 1e3
                if u in ("Gbyte",) and sc == 1e-6:
                    x *= 1e9
                vals.append("%.1f" % (x * sc) if sc != 1 or "%" in _ or m.startswith("gpu__time") else "%g" % x)
            except ValueError:
                vals.append(v)
        lines.append("| %s | %s | %s |" % (rep.split("/")[-1], d.get("Kernel Name", "?"), " | ".join(vals)))
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
