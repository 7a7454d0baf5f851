"""Generates tests/golden/ref_sketches.json: the REFERENCE's own emitted
CUDA kernels (pipeline.cpp run_codegen -> emitter.cpp generate_best_kernel,
compiled here from /root/reference/proj/src into oracle/_ref) for the six
reference fixtures and the SMALL bench configs, fused and unfused.

The reference never executes a graph, but its kernel sketches are complete
CUDA C: `tests/test_ref_sketches.py` compiles them for sm_100a, runs them on
a B200 and compares them with oracle/executor.py and with our executor --
that is what pins the numeric oracle to the reference.

Per case:
  * "fused":   the reference plan's selected patterns, plus a singleton
               pattern for every compute op the plan leaves unfused (the
               reference only emits kernels for fused ops), applied with the
               reference's apply_plan, then run_codegen;
  * "unfused": one singleton pattern per compute op (the one-kernel-per-op
               reference executor).
The graphs are restricted to the reference op set: a reduce carrying our
"name": "max" extension is emitted by the reference as a sum, so it is
stored here as a sum reduce (the oracle and our executor then evaluate the
same graph). Constant values travel with the graph; the reference takes
constants as kernel pointer arguments.

Run here (needs /root/reference and oracle/_ref): python scripts/make_ref_sketches.py
"""
import copy
import glob
import json
import re
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import refplan  # noqa: E402
from paper_1911_11576_b200 import workloads as W  # noqa: E402

FIX = "/root/reference/proj/fixtures"
COMPUTE = ("elementwise", "reduce", "dot", "batched_dot")


def reference_op_set(g):
    g = copy.deepcopy(g)
    for n in g["nodes"]:
        if n["kind"] == "reduce" and n.get("name") == "max":
            del n["name"]
    return g


def emits(g, pattern, limit):
    fused = refplan.call("apply_plan", graph=g, patterns=[pattern], selected=[0])["graph"]
    try:
        refplan.call("codegen", graph=fused, shared_limit_bytes=limit)
        return True
    except RuntimeError:
        return False


def split_emittable(g, pattern, limit):
    """Splits a pattern the reference cannot emit into maximal contiguous
    segments of its topological order that the reference does emit (a
    contiguous topo segment of a convex pattern is itself convex)."""
    order = [x for x in refplan.call("topo", graph=g) if x in set(pattern)]
    segs, cur = [], [order[0]]
    for x in order[1:]:
        if emits(g, cur + [x], limit):
            cur.append(x)
        else:
            segs.append(cur)
            cur = [x]
    return segs + [cur]


def sketches(g, patterns, limit, failed=None):
    """Reference kernels for `patterns`. A pattern the reference plans but its
    own emitter cannot emit ("no feasible template") is split into segments
    the reference does emit (split_emittable) and recorded in `failed` with
    the reference's reason."""
    patterns = [list(p) for p in patterns]
    while True:
        res = refplan.call("apply_plan", graph=g, patterns=patterns, selected=list(range(len(patterns))))
        fused = res["graph"]
        try:
            cg = refplan.call("codegen", graph=fused, shared_limit_bytes=limit)
            break
        except RuntimeError as e:
            m = re.match(r"no feasible template for (\S+): (.*)", str(e))
            if m is None or failed is None:
                raise
            node = next(n for n in fused["nodes"] if n["id"] == m.group(1))
            body = {b["id"] for b in node["body"]["nodes"] if b["kind"] in COMPUTE}
            i = next(i for i, p in enumerate(patterns) if set(p) == body)
            failed.append({"nodes": sorted(body), "reason": m.group(2)})
            segs = split_emittable(g, patterns[i], limit)
            failed[-1]["split_into"] = len(segs)
            patterns = patterns[:i] + segs + patterns[i + 1:]
    ks = []
    for m in cg["manifest"]["kernels"]:
        ks.append({"name": m["kernel"], "fused_op": m["fused_op"], "cta_num": m["cta_num"],
                   "cta_size": m["cta_size"], "shared_bytes": m["shared_bytes"],
                   "composition": m["composition"], "template": m["template"],
                   "source": cg["sources"][m["kernel"]]})
    return ks


def cases():
    for p in sorted(glob.glob(os.path.join(FIX, "*.json"))):
        yield "fixture:" + os.path.basename(p)[:-5], json.load(open(p))
    for name, fn in W.CONFIGS.items():
        yield name + "/small", fn(**W.SMALL[name])
    # A square LayerNorm: its row statistics [64] broadcast to [64, 64] map
    # onto the LAST dim under the IR's right-most-greedy rule (graph.cpp:158),
    # i.e. the graph means a column broadcast. The reference's fused kernel
    # reads the statistic for the CTA's own row instead (its block-scope value
    # cache ignores the broadcast map) -- a reference emitter inconsistency the
    # GPU test demonstrates; its unfused kernels follow the IR.
    yield "ambiguous:layernorm64x64", W.layernorm(rows=64, cols=64)


def main():
    out = []
    for name, g in cases():
        g = reference_op_set(g)
        ops = [n["id"] for n in g["nodes"] if n["kind"] in COMPUTE]
        t = time.time()
        entry = {"name": name, "graph": g, "variants": {}}
        entry["variants"]["unfused"] = sketches(g, [[o] for o in ops], W.REFERENCE_SHARED_LIMIT)
        for lim in (W.REFERENCE_SHARED_LIMIT, W.B200_SHARED_LIMIT):
            plan = refplan.call("plan", graph=g, shared_limit_bytes=lim)["plan"]
            pats = [plan["patterns"][i]["nodes"] for i in plan["selected"]]
            covered = {x for p in pats for x in p}
            pats += [[o] for o in ops if o not in covered]
            failed = []
            entry["variants"]["fused@%d" % lim] = sketches(g, pats, lim, failed)
            if failed:
                entry.setdefault("emit_failed", {})["fused@%d" % lim] = failed
        print("%-28s %s  %.1fs  emit_failed=%s" % (
            name, {k: len(v) for k, v in entry["variants"].items()}, time.time() - t,
            {k: len(v) for k, v in entry.get("emit_failed", {}).items()}), flush=True)
        out.append(entry)
    path = os.path.join(ROOT, "tests", "golden", "ref_sketches.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
