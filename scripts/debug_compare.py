"""Dev: run a config's bench plan and its unfused graph on the same inputs
and report outputs that differ (NaNs, max relative difference)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_11576_b200 import runtime as rt, tuning, workloads as W

name = sys.argv[1]
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = int(v)
torch.cuda.set_device(0)
g = W.CONFIGS[name](**kw)
plan = tuning.config_plan(name, g)[0]["fused"] if not kw else rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT, **W.PLAN_OPTIONS.get(name, {}))["fused"]
ex = rt.Executor(plan)
base = rt.Executor(g, chunking=False)
gen = torch.Generator(device="cuda"); gen.manual_seed(0)
ins = {t["id"]: torch.randn(t["dims"], device="cuda", generator=gen) for t in ex.info["inputs"]}
o1 = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
o2 = [torch.empty(t["dims"], device="cuda") for t in base.info["outputs"]]
ex.run([ins[i] for i in ex.input_ids], o1, stream=torch.cuda.current_stream().cuda_stream)
base.run([ins[i] for i in base.input_ids], o2, stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
names = base.output_ids
bad = 0
for n, a, b in zip(names, o1, o2):
    nan_a, nan_b = torch.isnan(a).sum().item(), torch.isnan(b).sum().item()
    d = ((a - b).abs() / (b.abs() + 1e-3)).max().item()
    if nan_a or nan_b or d > 1e-2:
        bad += 1
        if bad < 30:
            print("%-20s nan fused %d unfused %d  max rel diff %.3g" % (n, nan_a, nan_b, d))
print("outputs", len(names), "differing", bad)
k_of = {}
for k in ex.info["kernels"]:
    for o in k["outputs"]:
        k_of[o] = k["name"]
