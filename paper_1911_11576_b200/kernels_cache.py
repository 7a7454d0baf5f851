"""Build-time fill of the in-tree kernel cache (paper_1911_11576_b200/_kcache).

Every stitched kernel the benchmark and the GPU parity tests launch is
generated and compiled to an sm_100a cubin by NVRTC here (no GPU needed), so
the GPU box loads cubins instead of compiling. The cache is keyed by the
FNV-1a hash of the full kernel source plus the NVRTC options
(exec/runtime.cpp compile_cubin); a miss on the box just compiles there.
"""

from . import runtime as rt
from . import tuning
from . import workloads as W


def plans(full=True, small=True):
    """(tag, fused graph) for every plan bench.py and tests/ execute."""
    out = []
    for name, fn in W.CONFIGS.items():
        sizes = []
        if full:
            sizes.append(("full", {}))
        if small:
            sizes.append(("small", W.SMALL[name]))
        for size, kw in sizes:
            g = fn(**kw)
            if size == "full":
                out.append(("%s/%s/bench" % (name, size), tuning.config_plan(name, g)[0]["fused"]))
            if size == "full" and name in W.WHOLE_GRAPH:
                pass  # whole-graph config: only the (shipped) bench plan
            else:
                for lim_tag, lim in (("b200", W.B200_SHARED_LIMIT), ("ref48k", W.REFERENCE_SHARED_LIMIT)):
                    out.append(("%s/%s/%s" % (name, size, lim_tag), rt.plan(g, shared_limit_bytes=lim)["fused"]))
            out.append(("%s/%s/unfused" % (name, size), g))
    if full:
        # tests/test_executor_gpu.py: the bench BERT plan's groups at a 1024-token batch
        out.append(("bert/batch8/bench-groups", tuning.plan_like("bert", W.bert(batch=8))))
    return out


def _compile(args):
    fused_json, opts = args
    ex = rt.Executor(fused_json, compile_only=True, **opts)
    n = len(ex.info["kernels"])
    hits = sum(bool(k["cache_hit"]) for k in ex.info["kernels"])
    ex.close()
    return n, hits


def variant_jobs(configs=None):
    """(fused graph json, options) for every candidate of scripts/tune_variants.py."""
    import importlib.util
    import json
    import os
    spec = importlib.util.spec_from_file_location(
        "tv", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts", "tune_variants.py"))
    tv = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(tv)
    jobs = []
    for name in configs or list(W.CONFIGS):
        fused = json.dumps(tuning.config_plan(name)[0]["fused"])
        for v in tv.VARIANTS:
            jobs.append((fused, dict(v)))
    return jobs


def prebuild_variants(configs=None, workers=None):
    """Compile every tuning candidate (run before scripts/tune_variants.py on the box)."""
    import concurrent.futures as cf
    import os
    n = hits = 0
    with cf.ProcessPoolExecutor(workers or max(1, min(16, os.cpu_count() or 1))) as pool:
        for a, b in pool.map(_compile_safe, variant_jobs(configs)):
            n += a
            hits += b
    print("variant kernels: %d (%d already cached)" % (n, hits))


def _compile_safe(args):
    try:
        return _compile(args)
    except Exception:  # a variant that does not apply to a plan
        return 0, 0


def prebuild(verbose=True, workers=None):
    import concurrent.futures as cf
    import json
    import os
    jobs = []
    for tag, fused in plans():
        opts = {"chunking": False, "fold_constants": False, "sink_broadcasts": False} if tag.endswith("/unfused") else {}
        if tag.endswith("/bench") or tag.endswith("/bench-groups"):
            opts["kernel_options"] = tuning.kernel_variants(tag.split("/")[0])
        jobs.append((json.dumps(fused), opts))
        if tag.endswith("/unfused"):  # bench.py's folded unfused context line
            jobs.append((json.dumps(fused), {"chunking": False}))
    n = hits = 0
    with cf.ProcessPoolExecutor(workers or max(1, min(16, os.cpu_count() or 1))) as pool:
        for a, b in pool.map(_compile, jobs):
            n += a
            hits += b
    if verbose:
        print("kernel cache: %d kernels (%d already cached) in %s" % (n, hits, rt.CACHE_DIR))
