"""Dev: device time of chosen fused ops of a suite config's bench plan under
per-group codegen overrides, round-robin over the variants (L2 flushed before
every profiled pass; median of rounds x reps).
    python scripts/group_variants_ab.py bert fusion_5,fusion_38 '[{}, {"lazy_inputs": true}]' [rounds]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402

name, ops, variants = sys.argv[1], sys.argv[2].split(","), json.loads(sys.argv[3])
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 4
torch.cuda.set_device(0)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, device="cuda")
sink = torch.empty((), device="cuda")
fused = tuning.config_plan(name)[0]["fused"]
base = tuning.kernel_variants(name)
exs = []
for v in variants:
    ko = dict(base)
    for op in ops:
        ko[op] = v
    exs.append(rt.Executor(fused, kernel_options=ko))
ins = [torch.randn(t["dims"], device="cuda") for t in exs[0].info["inputs"]]
outs = [torch.empty(t["dims"], device="cuda") for t in exs[0].info["outputs"]]
acc = [{op: [] for op in ops} for _ in variants]
for _ in range(rounds):
    for vi, ex in enumerate(exs):
        for _ in range(3):
            with torch.cuda.stream(s):
                flush.zero_()
                torch.sum(rd, 0, out=sink)
            p = ex.profile(ins, outs, stream=s.cuda_stream, iters=1)
            for k in p["kernels"]:
                if k["op"] in acc[vi]:
                    acc[vi][k["op"]].append(k["us"])
for v, ex, a in zip(variants, exs, acc):
    info = {k["op"]: k for k in ex.info["kernels"]}
    print("%-80s %s" % (json.dumps(v)[:80], "  ".join("%s %.2f us (%s, blk %d grid %d)" % (
        op, float(np.median(a[op])), info[op]["scheme"].split("(")[0], info[op]["block"], info[op]["grid"]) for op in ops)),
          flush=True)
