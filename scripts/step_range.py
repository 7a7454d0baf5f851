"""One BERT (or any config) plan replay bracketed by cuProfilerStart/Stop, so
ncu's range replay reports the whole step's DRAM traffic and duration:
    ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python scripts/step_range.py bert '{"concurrent_lanes": 3}'
(never a timing source: ncu serialises and replays)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert"
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
torch.cuda.set_device(0)
opts.setdefault("kernel_options", tuning.kernel_variants(name))
fused = tuning.config_plan(name)[0]["fused"]
ex = rt.Executor(fused, **opts)
ins = [torch.randn(t["dims"], device="cuda") for t in ex.info["inputs"]]
outs = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(2):  # capture + warm the graph
    ex.run(ins, outs, stream=s.cuda_stream)
torch.cuda.synchronize()
with torch.cuda.stream(s):
    flush.zero_()
torch.cuda.synchronize()
torch.cuda.profiler.start()
ex.run(ins, outs, stream=s.cuda_stream)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("algo bytes per step", sum(k["algo_bytes"] for k in ex.info["kernels"]))
