"""Top stall SASS lines of an ncu report (--page source --print-source sass):
python scripts/ncu_hot.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
tot = sum(int(r[si]) for r in data if r[si].isdigit())
agg = {}
for r in data:
    for i in stall_cols:
        if r[i].isdigit():
            agg[h[i]] = agg.get(h[i], 0) + int(r[i])
print("total samples", tot)
print("by reason:", ", ".join("%s %.1f%%" % (k[6:], 100.0 * v / tot) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
for k, r in sorted(enumerate(data), key=lambda x: -(int(x[1][si]) if x[1][si].isdigit() else 0))[:n]:
    reasons = sorted(((int(r[i]) if r[i].isdigit() else 0, h[i][6:]) for i in stall_cols), reverse=True)[:2]
    print("%5s %5d %-70s %s" % (r[si], k, r[1].strip()[:70], reasons))
