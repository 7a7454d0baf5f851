"""A/B of whole-plan device time under executor option sets (graph replay,
L2 flushed before each pass, CUDA events, median of 15):
    python scripts/step_ab.py bert '[{}, {"colred_cluster": 0}]'
Each option set is applied on top of the shipped per-group variant table."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402

name = sys.argv[1]
variants = json.loads(sys.argv[2])
torch.cuda.set_device(0)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, device="cuda")
sink = torch.empty((), device="cuda")
fused = tuning.config_plan(name)[0]["fused"]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
exs = []
for v in variants:
    opts = dict(v)
    opts.setdefault("kernel_options", tuning.kernel_variants(name))
    exs.append(rt.Executor(fused, **opts))
ins = [torch.randn(t["dims"], device="cuda") for t in exs[0].info["inputs"]]
outs = [torch.empty(t["dims"], device="cuda") for t in exs[0].info["outputs"]]
times = [[] for _ in variants]
# round-robin: every variant measured in every round (drift hits all alike)
for rnd in range(rounds):
    # rotate the order every round: the variant measured first after a
    # switch runs slower (seen as a ~2 us penalty on a 72 us kernel)
    for vi in [(rnd + j) % len(exs) for j in range(len(exs))]:
        ex = exs[vi]
        for it in range(8):
            with torch.cuda.stream(s):
                flush.zero_()
                torch.sum(rd, 0, out=sink)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                ex.run(ins, outs, stream=s.cuda_stream)
                b.record(s)
            torch.cuda.synchronize()
            if it >= 2:
                times[vi].append(a.elapsed_time(b))
for v, ex, ts in zip(variants, exs, times):
    print("%-60s %3d kernels  median %.4f ms  min %.4f ms  (n=%d)" % (json.dumps(v)[:60], len(ex.info["kernels"]),
                                                                    float(np.median(ts)), min(ts), len(ts)), flush=True)
