"""Dev: device time of a fused graph JSON file under executor options
(L2 flushed before each pass; median of 10). Args: path[@key=json,key=json]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, device="cuda")
sink = torch.empty((), device="cuda")


def time_exec(fused, **opts):
    ex = rt.Executor(fused, **opts)
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
    return med, by / med / 1e3, [(k["name"], k["scheme"]) for k in ex.info["kernels"]]


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        path, _, opt = arg.partition("@")
        fused = json.load(open(path))
        opts = {}
        for kv in filter(None, opt.split(",")):
            k, v = kv.split("=")
            opts[k] = json.loads(v)
        med, gbs, ks = time_exec(fused, **opts)
        print("%-40s %-45s %8.1f us %6.0f GB/s %s" % (os.path.basename(path), json.dumps(opts), med, gbs, ks), flush=True)
