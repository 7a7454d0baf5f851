"""Reference-planner outputs for the execution-based plans of the bench
configs (the shipped B200 kernel-time CSVs fed to the reference's
CsvExecutionEvaluator) -> tests/golden/plans_exec.json. The CSV is referenced
by config name (paper_1911_11576_b200/data/b200_kernel_times/<name>.csv).
The encoder case takes the reference ~15 minutes."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import refplan  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402
from make_golden import strip  # noqa: E402

out = []
for name in W.CONFIGS:
    csv = tuning.load(name)
    if csv is None:
        continue
    t = time.time()
    res = refplan.call("plan", graph=W.CONFIGS[name](), mode="execution", kernel_times_csv=csv)
    print(name, "%.1fs" % (time.time() - t), flush=True)
    out.append({"name": name, "options": {"mode": "execution"}, "csv_config": name, "result": strip(res),
                "ref_seconds": round(time.time() - t, 1)})
with open(os.path.join(ROOT, "tests", "golden", "plans_exec.json"), "w") as f:
    json.dump(out, f, separators=(",", ":"))
print("wrote", len(out))
