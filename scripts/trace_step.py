"""Timeline of one plan pass from %globaltimer stamps (codegen option
`trace`; Executor.trace): per-kernel [start, end], concurrency, idle time.
    python scripts/trace_step.py bert '[{"concurrent_lanes": 1}, {"concurrent_lanes": 3}]' [--compile-only]
Writes gpurun_out/trace_<config>_<i>.json. The traced kernels carry two
extra atomics per warp; the span is close to, not equal to, the bench step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402

name = sys.argv[1]
variants = json.loads(sys.argv[2])
compile_only = "--compile-only" in sys.argv
fused = tuning.config_plan(name)[0]["fused"]
if not compile_only:
    import torch
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for vi, v in enumerate(variants):
    opts = dict(v, trace=True)
    opts.setdefault("kernel_options", tuning.kernel_variants(name))
    ex = rt.Executor(fused, compile_only=compile_only, **opts)
    if compile_only:
        continue
    ins = [torch.randn(t["dims"], device="cuda") for t in ex.info["inputs"]]
    outs = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
    for _ in range(3):
        ex.run(ins, outs, stream=s.cuda_stream)
    spans = []
    best = None
    for _ in range(5):
        with torch.cuda.stream(s):
            flush.zero_()
        tr = ex.trace(ins, outs, stream=s.cuda_stream)
        spans.append(tr["span_us"])
        if best is None or tr["span_us"] < best["span_us"]:
            best = tr
    ks = best["kernels"]
    ev = sorted([(k["start_us"], 1) for k in ks] + [(k["end_us"], -1) for k in ks])
    busy = {}
    cur, last = 0, 0.0
    for t, d in ev:
        busy[cur] = busy.get(cur, 0.0) + t - last
        cur += d
        last = t
    dur = sum(k["end_us"] - k["start_us"] for k in ks)
    print("%s %s: span %.1f us (runs %s), sum of kernel durations %.1f us, time at concurrency %s" % (
        name, json.dumps(v), best["span_us"], [round(x, 1) for x in spans], dur,
        {c: round(t, 1) for c, t in sorted(busy.items())}), flush=True)
    top = sorted(ks, key=lambda k: k["start_us"] - k["end_us"])[:12]
    for k in top:
        d = k["end_us"] - k["start_us"]
        print("   %-14s %7.2f us  %6.0f GB/s  [%7.1f, %7.1f]" % (k["name"], d, k["algo_bytes"] / d / 1e3, k["start_us"], k["end_us"]))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/trace_%s_%d.json" % (name, vi), "w") as f:
        json.dump(dict(options=v, spans=spans, **best), f)
