"""Per-group kernel selection (paper Alg. 3 KernelEvalUpdate; reference
emitter.cpp:1346 select_best / :1367 generate_best_kernel with a
KernelEvaluator, emitter.hpp:153): every fused op of a suite config's bench
plan is generated under each codegen variant below, each candidate kernel is
timed on the GPU (stitch_executor_profile: CUDA events around the launch on
its stream, L2 flushed before every pass, median of --reps), and the fastest
is kept per fused op -- the default unless a variant is faster by more than
--min-gain. Writes paper_1911_11576_b200/data/kernel_variants/<config>.json
({op id: codegen overrides}, plus the measurements), which tuning.py feeds to
the executor as `kernel_options`.

    python scripts/tune_variants.py bert [--reps 5]      (on a B200)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1911_11576_b200 import tuning  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402

# candidate implementations per fused op (options that change the generated kernel)
VARIANTS = [
    {},
    {"wide_cross_cta": True},
    {"wide_cross_cta": True, "wide_cross_threads": 128},
    {"wide_cross_cta": True, "wide_cross_threads": 384},
    {"wide_cross_cta": True, "wide_cross_threads": 192},
    {"wide_cross_cta": True, "wide_cross_threads": 256},
    {"lazy_inputs": True, "cross_smem": False},
    {"cross_smem": False},
    {"row_prefetch_warp": True},
    {"row_prefetch": False},
    {"lazy_inputs": True},
    {"loop_fusion": False},
    {"colred_cols": 64},
    {"colred_cols": 128},
    {"colred_cluster": 8},
    {"colred_cluster": 0},
    {"colred_eout": True},
    {"colred_eout": True, "colred_cluster": 0},
    {"colred_eout": True, "colred_cols": 128},
    {"pack_sequential": True},
    {"tma_double_buffer": True},
    {"nr_divide": True},
    {"min_ctas_per_sm": 3},
    {"min_ctas_per_sm": 2},
    {"nr_divide": True, "min_ctas_per_sm": 3},
    {"nr_divide": True, "loop_fusion": False},
    {"nr_divide": True, "wide_cross_cta": True, "wide_cross_threads": 192},
    {"narrow_rows": False},
    {"cta_rows": 128},
    {"cta_rows": 192},
    {"cta_rows": 256},
    {"cta_rows": 192, "loop_fusion": False},
    {"cta_threads": 128},
    {"cta_threads": 384},
    {"cta_threads": 512},
    {"cta_threads": 768},
    {"cta_rows": 64},
    {"cta_rows": 96},
    {"cta_threads": 192},
    {"cta_rows": 192, "lazy_inputs": True},
    {"cta_rows": 128, "lazy_inputs": True},
    {"cta_rows": 256, "lazy_inputs": True},
    {"cta_threads": 384, "lazy_inputs": True},
    {"cta_rows": 192, "min_ctas_per_sm": 2},
]
# Not candidates: split_cross (one kernel + grid barrier instead of a row
# kernel and its fold). Timed alone the single kernel wins, inside the
# dataflow step the split wins (its fold leaves the critical path: BERT
# 1.732 -> 1.602 ms), so it is decided on the whole step, not per kernel.


def main():
    import torch
    from paper_1911_11576_b200 import runtime as rt
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--min-gain", type=float, default=0.03)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rd = torch.ones(64 << 20, device="cuda")
    sink = torch.empty((), device="cuda")

    def flush_l2():
        with torch.cuda.stream(s):
            flush.zero_()
            torch.sum(rd, 0, out=sink)

    g = W.CONFIGS[a.config]()
    fused = tuning.config_plan(a.config, g)[0]["fused"]
    times = {}  # variant index -> {op: us}
    ins = outs = None
    for vi, v in enumerate(VARIANTS):
        t0 = time.time()
        try:
            ex = rt.Executor(fused, **v)
        except rt.StitchError as e:
            print("variant %s: %s" % (v, str(e).splitlines()[0]), flush=True)
            continue
        if ins is None:
            gen = torch.Generator(device="cuda")
            gen.manual_seed(5)
            ins = [torch.randn(t["dims"], device="cuda", generator=gen) for t in ex.info["inputs"]]
            outs = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
        acc = {}
        for _ in range(a.reps):
            flush_l2()
            prof = ex.profile(ins, outs, stream=s.cuda_stream, iters=1)
            per_op = {}  # a split row group's row kernel + fold count together
            for k in prof["kernels"]:
                op = k["op"] if "op" in k else k["name"]
                per_op[op] = per_op.get(op, 0.0) + k["us"]
            for op, us in per_op.items():
                acc.setdefault(op, []).append(us)
        times[vi] = {op: float(np.median(us)) for op, us in acc.items()}
        print("variant %-55s total %8.1f us  (%.0f s)" % (json.dumps(v), sum(times[vi].values()), time.time() - t0),
              flush=True)
        ex.close()
    base = times[0]
    table, chosen = {}, {}
    for op, t_def in base.items():
        best_v, best_t = 0, t_def
        for vi, tv in times.items():
            if op in tv and tv[op] < best_t:
                best_v, best_t = vi, tv[op]
        if best_v and best_t < t_def * (1 - a.min_gain):
            table[op] = VARIANTS[best_v]
        chosen[op] = {"default_us": round(t_def, 2), "best_us": round(best_t if best_v and best_t < t_def * (1 - a.min_gain)
                                                                        else t_def, 2),
                      "variant": VARIANTS[best_v] if op in table else {}}

    def step_once(ex):
        flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ex.run(ins, outs, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    ex0 = rt.Executor(fused)
    ex1 = rt.Executor(fused, kernel_options=table)
    t0s, t1s = [], []
    for i in range(30):  # alternating, so clock / thermal drift hits both
        t0s.append(step_once(ex0))
        t1s.append(step_once(ex1))
    step0, step1 = float(np.median(t0s[5:])), float(np.median(t1s[5:]))
    print("step: default %.4f ms, tuned %.4f ms (%d of %d groups changed)" % (step0, step1, len(table), len(base)))
    all_times = {op: {str(vi): round(tv[op], 2) for vi, tv in times.items() if op in tv} for op in base}
    res = {"config": a.config, "plan_signature": tuning.plan_signature(fused), "variants": VARIANTS, "table": table,
           "per_op": chosen, "times_us": all_times,
           "step_ms": {"default": step0, "tuned": step1}, "reps": a.reps, "min_gain": a.min_gain}
    out = a.out or os.path.join(ROOT, "paper_1911_11576_b200", "data", "kernel_variants", a.config + ".json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
