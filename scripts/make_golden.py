"""Generates tests/golden/plans.json from the REFERENCE planner
(oracle/_ref/libstitch_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run here, where the reference exists; the committed output
lets tests/test_golden.py check plan parity on machines without it.

Each entry: {"name", "graph", "options", "result"}; `result` is the
reference's run_plan output (plan.json, fused graph, report text).
The reference fixtures (proj/fixtures/*.json) are small test inputs and are
embedded verbatim as `graph`.
"""
import glob
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import refplan  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402

FIX = "/root/reference/proj/fixtures"


def cases(full):
    for p in sorted(glob.glob(os.path.join(FIX, "*.json"))):
        g = json.load(open(p))
        for lim in (W.REFERENCE_SHARED_LIMIT, W.B200_SHARED_LIMIT):
            yield "fixture:%s@%d" % (os.path.basename(p)[:-5], lim), g, {"shared_limit_bytes": lim}
        yield "fixture:%s@substitution" % os.path.basename(p)[:-5], g, {"strategy": "substitution"}
    for name, fn in W.CONFIGS.items():
        # whole-graph configs (W.WHOLE_GRAPH) are beyond the reference's search at full size
        sizes = [("small", W.SMALL[name])] + ([("full", {})] if full and name not in W.WHOLE_GRAPH else [])
        for size, kw in sizes:
            g = fn(**kw)
            for lim in (W.REFERENCE_SHARED_LIMIT, W.B200_SHARED_LIMIT):
                yield "%s/%s@%d" % (name, size, lim), g, {"shared_limit_bytes": lim}


def strip(x):
    if isinstance(x, dict):
        return {k: strip(v) for k, v in x.items() if k not in ("value", "timings")}
    if isinstance(x, list):
        return [strip(v) for v in x]
    return x


def main():
    full = "--full" in sys.argv
    out = []
    for name, g, opts in cases(full):
        t = time.time()
        res = refplan.call("plan", graph=g, **opts)
        print("%-40s %.1fs" % (name, time.time() - t), flush=True)
        out.append({"name": name, "graph": g, "options": opts, "result": strip(res),
                    "ref_seconds": round(time.time() - t, 2)})
    path = os.path.join(ROOT, "tests", "golden", "plans_full.json" if full else "plans.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"), sort_keys=False)
    print("wrote", path, len(out), "cases")


if __name__ == "__main__":
    main()
