"""Quick GPU bring-up check: every config (small + full), fused (both shared
limits) and unfused, against the CPU oracle; prints errors and kernel times."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1911_11576_b200 import runtime as rt, workloads as W
from oracle import executor as orc

SMALL = {
    "layernorm": dict(rows=256, cols=768),
    "softmax": dict(heads=2, seq=128),
    "encoder": dict(batch=2, seq=64, hidden=1024),
    "gru": dict(batch=64, n=64),
}

def check(name, g, fused, tag, full):
    ex = rt.Executor(fused)
    ins = orc.random_inputs(g, seed=1)
    tin = [torch.from_numpy(ins[i]).cuda() for i in ex.input_ids]
    outs = [torch.empty(t["dims"], dtype=torch.float32, device="cuda") for t in ex.info["outputs"]]
    ex.run(tin, outs)
    torch.cuda.synchronize()
    ref = orc.run(g, ins)
    worst = 0.0
    for o, r in zip(outs, ref):
        d = np.abs(o.cpu().numpy().astype(np.float64) - r.astype(np.float64))
        tol = np.maximum(1e-5 * np.abs(r), 1e-6)
        worst = max(worst, float((d / tol).max()))
    prof = ex.profile(tin, outs, iters=5)
    print(f"{name:10s} {tag:8s} full={full} kernels={len(ex.info['kernels'])} err/tol={worst:.3g} total_us={prof['total_us']:.1f} "
          + " ".join(f"{k['name']}:{k['us']:.1f}us/{k['gbps']:.0f}GBs" for k in prof['kernels'][:6]), flush=True)

for name, fn in W.CONFIGS.items():
    for full in (False, True):
        g = fn() if full else fn(**SMALL[name])
        for tag, lim in (("b200", 232448), ("ref48k", 49152)):
            p = rt.plan(g, shared_limit_bytes=lim)
            try:
                check(name, g, p["fused"], tag, full)
            except Exception as e:
                print(name, tag, full, "FAILED", repr(e)[:2000], flush=True)
        try:
            check(name, g, g, "unfused", full)
        except Exception as e:
            print(name, "unfused", full, "FAILED", repr(e)[:2000], flush=True)
