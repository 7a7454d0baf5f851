"""Dev sweep: device time of each config's fused plan under executor
options (chunking, pipelining, chunk sizes), L2 flushed before each pass,
CUDA events on the launching stream, median of N passes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402

VARIANTS = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [
    {"chunking": False}, {"chunk_pipeline": False}, {}, {"chunk_l2_bytes": 8 << 20}, {"chunk_l2_bytes": 4 << 20},
    {"chunk_l2_bytes": 8 << 20, "chunk_ring": 3}]
CONFIGS = sys.argv[2].split(",") if len(sys.argv) > 2 else list(W.CONFIGS)
torch.cuda.set_device(0)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, device="cuda")
sink = torch.empty((), device="cuda")
for name in CONFIGS:
    g = W.CONFIGS[name]()
    fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    for v in VARIANTS:
        ex = rt.Executor(fused, **v)
        ins = [torch.randn(t["dims"], device="cuda") for t in ex.info["inputs"]]
        outs = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
        ts = []
        for it in range(12):
            with torch.cuda.stream(s):
                flush.zero_()
                torch.sum(rd, 0, out=sink)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                ex.run(ins, outs, stream=s.cuda_stream)
                b.record(s)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(a.elapsed_time(b) * 1e3)
        by = sum(t["bytes"] for t in ex.info["inputs"]) + sum(t["bytes"] for t in ex.info["outputs"])
        med = float(np.median(ts))
        print("%-9s %-55s %8.1f us  %6.0f GB/s  sched=%s" % (name, json.dumps(v), med, by / med / 1e3,
              [(x["kernels"], x["chunks"]) for x in ex.info["schedule"]]), flush=True)
        ex.close()
