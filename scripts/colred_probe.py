"""Dev probe: a lone [R, C] column sum through the executor under COLRED
options; per-launch device time from a 20-launch CUDA-graph replay (L2
flushed before the replay) and from stitch_executor_profile."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402

R, C = int(sys.argv[1]), int(sys.argv[2])
variants = json.loads(sys.argv[3]) if len(sys.argv) > 3 else [{}]
g = {"nodes": [{"id": "x", "kind": "parameter", "shape": {"dims": [R, C], "dtype": "f32"}},
               {"id": "s", "kind": "reduce", "operands": ["x"], "reduce_dims": [0], "shape": {"dims": [C], "dtype": "f32"}}],
     "outputs": ["s"]}
torch.cuda.set_device(0)
x = torch.randn(R, C, device="cuda")
o = torch.empty(C, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
for v in variants:
    ex = rt.Executor(g, **v)
    k = ex.info["kernels"][0]
    ts = []
    for rep in range(5):
        with torch.cuda.stream(st):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            ex.run([x], [o], stream=st.cuda_stream)
            b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    # warm (L2-resident input) back-to-back
    with torch.cuda.stream(st):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(20):
            ex.run([x], [o], stream=st.cuda_stream)
        b.record(st)
    torch.cuda.synchronize()
    warm = a.elapsed_time(b) * 1e3 / 20
    ref = x.double().sum(0).float()
    err = (o - ref).abs().max().item()
    print("%-40s %-28s grid %4d block %3d smem %6d: cold %.2f us (min %.2f), warm b2b %.2f us, %.0f GB/s cold; err %.2e" % (
        json.dumps(v), k["scheme"], k["grid"], k["block"], k["smem_bytes"], sorted(ts)[2], min(ts), warm,
        R * C * 4 / (sorted(ts)[2] * 1e3), err), flush=True)
