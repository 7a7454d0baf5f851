"""Execution-based pattern scoring on B200 (paper §4.3; reference
cost_model.cpp score_execution_based, pipeline.cpp CsvExecutionEvaluator).

The reference scores a fusion pattern P either with the bandwidth model,
f(P) = M(V) + (N-1)·φ, gated by its shared-memory sketch model, or -- "for
complex ones", and for all of them in ExecutionBased mode -- by measured
kernel times, f(P) = Σ K(op_j) + (N-1)·φ − K(P). Its evaluator is a
pluggable interface fed from a `name,kernel_us` CSV. Here the stitched
executor is that evaluator: every candidate pattern the planner generates is
compiled into its stitched sm_100a kernel and timed on the GPU (L2 flushed
before every timing, median of `iters`), and so is every op as its own
kernel. The CSV is then handed to the planner (`kernel_times_csv` with
`mode: "execution"`), which runs the reference's exact selection (ILP with
cycle elimination) on the measured scores -- the same CSV gives the same plan
in the reference planner, bit for bit.

    csv = tuning.measure(graph)                       # on a B200
    plan = runtime.plan(graph, mode="execution", kernel_times_csv=csv)

Measured tables for the bench configs ship in
paper_1911_11576_b200/data/b200_kernel_times/<config>.csv.
"""

import concurrent.futures as cf
import hashlib
import json
import os

from . import runtime as rt

DATA_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "b200_kernel_times")


def pattern_graph(graph, nodes):
    """A graph holding only pattern `nodes` fused into one op (its external
    operands become parameters; scalar constants stay literals)."""
    r = rt.debug_call("apply_plan", graph=graph, patterns=[sorted(nodes)], selected=[0])
    fg = r["graph"]
    by_id = {n["id"]: n for n in fg["nodes"]}
    fused = next(n for n in fg["nodes"] if n["kind"] == "fused")
    out, seen = [], set()
    for o in fused["operands"]:
        if o in seen:
            continue
        seen.add(o)
        src = by_id[o]
        if src["kind"] == "constant":
            out.append(src)
        else:
            out.append({"id": o, "kind": "parameter", "shape": src["shape"]})
    return {"nodes": out + [fused], "outputs": [fused["id"]]}


def fused_key(nodes):
    """Row name of a pattern in the CSV: op ids in std::set<std::string>
    order joined by '+' (pipeline.cpp CsvExecutionEvaluator::measure)."""
    return "+".join(sorted(nodes, key=lambda s: s.encode()))


def candidate_patterns(graph, **plan_options):
    keys = ("strategy", "max_operands", "seed_min_bytes", "exploration_budget", "large_dot_flops")
    return rt.debug_call("generate_patterns", graph=graph, **{k: v for k, v in plan_options.items() if k in keys})


def _compile_one(args):
    g_json, opts = args
    ex = rt.Executor(g_json, compile_only=True, **opts)
    n = len(ex.info["kernels"])
    ex.close()
    return n


def precompile(graph, workers=None, exec_options=None, **plan_options):
    """Compile (NVRTC, no GPU) the kernel of every candidate pattern and of
    every op into the kernel cache, in parallel."""
    opts = dict(exec_options or {})
    jobs = [(json.dumps(graph), dict(opts, chunking=False))]
    for p in candidate_patterns(graph, **plan_options):
        jobs.append((json.dumps(pattern_graph(graph, p["nodes"])), opts))
    with cf.ProcessPoolExecutor(workers or os.cpu_count()) as pool:
        return sum(pool.map(_compile_one, jobs, chunksize=8))


def _time_executor(ex, iters, torch, flush):
    d_in = [torch.randn(t["dims"], device="cuda") for t in ex.info["inputs"]]
    d_out = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
    stream = torch.cuda.current_stream().cuda_stream
    ex.run(d_in, d_out, stream=stream)  # warm-up (module load, first touch)
    samples = {}
    for _ in range(iters):
        flush()
        prof = ex.profile(d_in, d_out, stream=stream, iters=1)
        for k in prof["kernels"]:
            samples.setdefault(k["op"], []).append(k["us"])
    return {op: sorted(v)[len(v) // 2] for op, v in samples.items()}


def measure(graph, iters=5, device=0, exec_options=None, progress=False, **plan_options):
    """Measured kernel times of every op and every candidate pattern of
    `graph` on `device`, as the reference's `name,kernel_us` CSV text."""
    import torch

    torch.cuda.set_device(device)
    junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rd = torch.ones(64 << 20, device="cuda")
    sink = torch.empty((), device="cuda")

    def flush():
        junk.zero_()
        torch.sum(rd, 0, out=sink)

    opts = dict(exec_options or {})
    rows = []
    ex = rt.Executor(graph, device=device, chunking=False, **opts)
    per_op = _time_executor(ex, iters, torch, flush)
    ex.close()
    for op in sorted(per_op, key=lambda s: s.encode()):
        rows.append((op, per_op[op]))
    pats = candidate_patterns(graph, **plan_options)
    for i, p in enumerate(pats):
        pg = pattern_graph(graph, p["nodes"])
        ex = rt.Executor(pg, device=device, **opts)
        t = _time_executor(ex, iters, torch, flush)
        ex.close()
        fused_id = pg["outputs"][0]
        rows.append((fused_key(p["nodes"]), t[fused_id]))
        if progress and i % 100 == 0:
            print("  measured %d/%d patterns" % (i + 1, len(pats)), flush=True)
    lines = ["name,kernel_us"] + ["%s,%.4f" % (n, us) for n, us in rows]
    return "\n".join(lines) + "\n"


def load(config):
    """The shipped B200 kernel-time table of bench config `config`, or None."""
    p = os.path.join(DATA_DIR, config + ".csv")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return f.read()


PLAN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "plans")


def _plan_key(graph, options):

    blob = json.dumps({"graph": graph, "options": options}, sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(blob.encode()).hexdigest()


def cached_plan(name, graph, options):
    """Shipped plan of `graph` under `options` (data/plans/<name>.json), used
    when the key (sha256 of graph + options) matches -- planning the 12-layer
    BERT graph takes minutes; scripts/make_plan_cache.py recomputes it with
    stitch_plan_graph and checks it is reproduced exactly. None on a miss."""
    p = os.path.join(PLAN_DIR, name + ".json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    if d.get("key") != _plan_key(graph, options):
        return None
    return d["result"]


def kernel_variants(name, fused=None):
    """The measured per-group codegen variant table of suite config `name`
    (data/kernel_variants/<name>.json, scripts/tune_variants.py): {op id:
    codegen overrides}, passed to the executor as kernel_options; {} when
    none is shipped, or when it was measured on another plan (its
    `plan_signature` differs from that of `fused`, default: the plan bench.py
    runs) -- op ids name different groups then."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "kernel_variants", name + ".json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        d = json.load(f)
    if fused is None:
        fused = config_plan(name)[0]["fused"]
    if d.get("plan_signature") != plan_signature(fused):
        import warnings
        warnings.warn("kernel variant table %s was measured on another plan; not used" % p)
        return {}
    return d["table"]


def plan_signature(fused):
    """Identity of a fused graph's grouping (sha256 of its fusion groups)."""
    return hashlib.sha256(json.dumps(groups_of(fused)).encode()).hexdigest()[:16]


def groups_of(fused):
    """The fusion groups (op ids per fused node) of a fused graph."""
    return [[m["id"] for m in n["body"]["nodes"] if m["kind"] not in ("parameter", "tuple", "constant")]
            for n in fused["nodes"] if n["kind"] == "fused"]


def plan_like(name, graph):
    """`graph` (the config at another batch size: op ids do not depend on it)
    fused with exactly the groups of the plan bench.py runs for `name` --
    e.g. the shipped 12-layer BERT plan at a batch the oracle can check."""
    fused = config_plan(name)[0]["fused"]
    pats = groups_of(fused)
    return rt.debug_call("apply_plan", graph=graph, patterns=pats, selected=list(range(len(pats))))["graph"]


def config_plan(name, graph=None, shared_limit_bytes=None):
    """The plan bench.py runs for suite config `name`: execution-based scores
    from the shipped B200 table when `graph` is the config at its BASELINE
    size (the table is keyed by op ids measured at that size), else the
    model-based plan at the B200 shared-memory limit. Returns
    (plan result, description)."""
    from . import workloads as W
    if graph is None:
        graph = W.CONFIGS[name]()
    csv = load(name)
    if csv is not None and graph == W.CONFIGS[name]():
        return rt.plan(graph, mode="execution", kernel_times_csv=csv), "execution-based (B200-measured kernel times)"
    lim = shared_limit_bytes or W.B200_SHARED_LIMIT
    opts = dict({"shared_limit_bytes": lim}, **W.PLAN_OPTIONS.get(name, {}))
    hit = cached_plan(name, graph, opts)
    if hit is not None:
        return hit, "model-based (T=%d B), shipped plan" % lim
    return rt.plan(graph, **opts), "model-based (T=%d B)" % lim
