"""Runs every suite config's fused plan (and optionally the unfused
baseline) a few times with plain launches -- the command ncu wraps for the
launch list and the --set full captures (never a timing source)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default=",".join(W.CONFIGS))
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--unfused", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
for name in a.configs.split(","):
    g = W.CONFIGS[name]()
    graphs = [("fused", tuning.config_plan(name, g)[0]["fused"])]
    if a.unfused:
        graphs.append(("unfused", g))
    for tag, fg in graphs:
        ex = rt.Executor(fg, use_graph=False, **({"kernel_options": tuning.kernel_variants(name)} if tag == "fused" else {"fold_constants": False, "sink_broadcasts": False}))
        ins = [torch.randn(t["dims"], device="cuda") for t in ex.info["inputs"]]
        outs = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
        for _ in range(a.iters):
            ex.run(ins, outs, stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        seq = [k for s in ex.info["schedule"] for _ in range(s["chunks"]) for k in s["kernels"]]
        print(name, tag, seq, flush=True)
