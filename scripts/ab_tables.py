"""A/B of whole-step device time between per-group variant tables (graph
replay, L2 flushed before each pass, CUDA events, alternating rounds):
    python scripts/ab_tables.py bert table_a.json table_b.json [rounds]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402

name, files = sys.argv[1], [a for a in sys.argv[2:] if a.endswith(".json")]
rounds = int(sys.argv[-1]) if not sys.argv[-1].endswith(".json") else 6
torch.cuda.set_device(0)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, device="cuda")  # read after the flush: no dirty lines left in L2
sink = torch.empty((), device="cuda")
fused = tuning.config_plan(name)[0]["fused"]
exs = [rt.Executor(fused, kernel_options=json.load(open(f))["table"]) for f in files]
ins = [torch.randn(t["dims"], device="cuda") for t in exs[0].info["inputs"]]
outs = [torch.empty(t["dims"], device="cuda") for t in exs[0].info["outputs"]]
times = [[] for _ in files]
for rnd in range(rounds):
    for i in [(rnd + j) % len(exs) for j in range(len(exs))]:  # rotated: no first-after-switch bias
        ex = exs[i]
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
                times[i].append(a.elapsed_time(b))
for f, ts in zip(files, times):
    print("%-50s median %.4f ms  min %.4f ms" % (f, float(np.median(ts)), min(ts)))
