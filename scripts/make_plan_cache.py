"""Plans a suite config with stitch_plan_graph (model-based, T = 227 KiB)
twice, checks the two results are identical, and ships the plan as
paper_1911_11576_b200/data/plans/<config>.json keyed by sha256(graph +
options) (tuning.cached_plan)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402

name = sys.argv[1]
g = W.CONFIGS[name]()
opts = dict({"shared_limit_bytes": W.B200_SHARED_LIMIT}, **W.PLAN_OPTIONS.get(name, {}))
t = time.time()
a = rt.plan(g, **opts)
t1 = time.time() - t
b = rt.plan(g, **opts)
ta, tb = a.pop("timings"), b.pop("timings")
assert a == b, "planning is not deterministic"
assert ta["ilp_truncated"] == 0, "the selection search hit its node budget: plan not exact"
os.makedirs(tuning.PLAN_DIR, exist_ok=True)
# the candidate list (200k patterns) is not shipped: count + the selected ones
pl = a["plan"]
pl["patterns"] = {"count": len(pl["patterns"]), "selected": [pl["patterns"][i] for i in pl["selected"]]}
with open(os.path.join(tuning.PLAN_DIR, name + ".json"), "w") as f:
    json.dump({"key": tuning._plan_key(g, opts), "options": opts, "plan_seconds": round(t1, 1), "timings": ta,
               "result": a}, f, separators=(",", ":"))
groups = sum(1 for n in a["fused"]["nodes"] if n["kind"] == "fused")
print(name, "planned in %.1fs" % t1, "groups", groups, ta)
