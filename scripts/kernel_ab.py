"""Dev: per-kernel device times of a fused graph under two option sets
(L2 flushed before each profiled pass, median of 5); prints the largest
differences. Usage: kernel_ab.py graph.json key=val,... key=val,..."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_11576_b200 import runtime as rt

def parse(o):
    d = {}
    for kv in filter(None, o.split(",")):
        k, v = kv.split("=")
        d[k] = json.loads(v)
    return d

torch.cuda.set_device(0)
g = json.load(open(sys.argv[1]))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for o in sys.argv[2:4]:
    ex = rt.Executor(g, **parse(o))
    ins = [torch.randn(t["dims"], device="cuda") for t in ex.info["inputs"]]
    outs = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
    s = torch.cuda.current_stream().cuda_stream
    acc = {}
    for it in range(5):
        flush.zero_()
        p = ex.profile(ins, outs, stream=s, iters=1)
        for k in p["kernels"]:
            acc.setdefault(k["name"], []).append(k["us"])
    res.append({k: sorted(v)[2] for k, v in acc.items()})
    scheme = {k["name"]: k["scheme"] for k in ex.info["kernels"]}
    res[-1]["__scheme"] = scheme
a, b = res
print("total A %.1f us, B %.1f us" % (sum(v for k, v in a.items() if k != "__scheme"), sum(v for k, v in b.items() if k != "__scheme")))
diffs = sorted(((b[k] - a[k], k) for k in a if k != "__scheme"), reverse=True)
for d, k in diffs[:12] + diffs[-12:]:
    print("%-14s A %7.1f  B %7.1f  %s | %s" % (k, a[k], b[k], a["__scheme"][k][:40], b["__scheme"][k][:40]))
