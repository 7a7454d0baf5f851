"""Measures the execution-based scoring table of every bench config on a
B200 (paper_1911_11576_b200/tuning.py) and writes
gpurun_out/b200_kernel_times/<config>.csv; copy them into
paper_1911_11576_b200/data/b200_kernel_times/ to ship them."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_11576_b200 import tuning  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(W.CONFIGS)
out = os.path.join("gpurun_out", "b200_kernel_times")
os.makedirs(out, exist_ok=True)
for n in names:
    t = time.time()
    csv = tuning.measure(W.CONFIGS[n](), iters=5, progress=True)
    with open(os.path.join(out, n + ".csv"), "w") as f:
        f.write(csv)
    print(n, "rows", csv.count("\n") - 1, "%.1fs" % (time.time() - t), flush=True)
