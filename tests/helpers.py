"""Shared test helpers (random DAG generator, GPU run helper)."""
import random

import numpy as np

ELEM_BIN = ["add", "subtract", "multiply", "divide", "maximum", "minimum"]
ELEM_UN = ["exp", "negate", "log", "rsqrt"]


def random_dag(seed, n_ops=12, dims=(64, 256), reduce_p=0.2):
    """Seeded random graph in the reference JSON format over one 2-D shape:
    elementwise ops, row / column reductions and broadcasts back."""
    rng = random.Random(seed)
    R, C = dims
    nodes = [{"id": "p0", "kind": "parameter", "shape": {"dims": [R, C], "dtype": "f32"}},
             {"id": "p1", "kind": "parameter", "shape": {"dims": [R, C], "dtype": "f32"}}]
    full = ["p0", "p1"]
    for i in range(n_ops):
        nid = "n%02d" % i
        r = rng.random()
        if r < reduce_p:
            src = rng.choice(full)
            if rng.random() < 0.5:
                nodes.append({"id": nid + "r", "kind": "reduce", "operands": [src], "reduce_dims": [1],
                              "shape": {"dims": [R], "dtype": "f32"}})
            else:
                nodes.append({"id": nid + "r", "kind": "reduce", "operands": [src], "reduce_dims": [0],
                              "shape": {"dims": [C], "dtype": "f32"}})
            nodes.append({"id": nid, "kind": "elementwise", "name": "broadcast", "operands": [nid + "r"],
                          "shape": {"dims": [R, C], "dtype": "f32"}})
        elif r < 0.4:
            nodes.append({"id": nid, "kind": "elementwise", "name": rng.choice(["exp", "negate"]),
                          "operands": [rng.choice(full)], "shape": {"dims": [R, C], "dtype": "f32"}})
        else:
            a, b = rng.choice(full), rng.choice(full)
            nodes.append({"id": nid, "kind": "elementwise", "name": rng.choice(["add", "subtract", "multiply"]),
                          "operands": [a, b], "shape": {"dims": [R, C], "dtype": "f32"}})
        full.append(nid)
    consumed = {o for n in nodes for o in n.get("operands", [])}
    outs = [n["id"] for n in nodes if n["id"] not in consumed and n["kind"] != "parameter"]
    if not outs:
        outs = [full[-1]]
    return {"nodes": nodes, "outputs": outs}


def scaled_inputs(graph, seed=0, scale=0.5):
    from oracle import executor as orc
    return orc.random_inputs(graph, seed=seed, scale=scale)


def _node(i, k, ops=None, name=None, dims=(4096, 256), **kw):
    d = {"id": i, "kind": k, "shape": {"dims": list(dims), "dtype": "f32"}}
    if ops:
        d["operands"] = ops
    if name:
        d["name"] = name
    d.update(kw)
    return d


def chunk_chain_graph(R=4096, C=256):
    """exp -> multiply -> add (three chunkable kernels, unfused) feeding a
    column reduce that cannot be chunked."""
    return {"nodes": [_node("x", "parameter", dims=(R, C)),
                      _node("a", "elementwise", ["x"], "exp", dims=(R, C)),
                      _node("b", "elementwise", ["a", "x"], "multiply", dims=(R, C)),
                      _node("y", "elementwise", ["b", "x"], "add", dims=(R, C)),
                      _node("cs", "reduce", ["y"], dims=(C,), reduce_dims=[0])],
            "outputs": ["cs"]}



def contract_selection(scores, sets, cycles):
    """Brute force of the selection contract (reference
    proj/src/ilp_solver.cpp:139 solve, small k only): optimum = max over
    node-disjoint selections within the cycle limits of the ascending-order
    double sum; answer = the index-by-index lexicographic extraction
    (ilp_solver.cpp:153-167)."""
    k = len(scores)
    optimal, opt = [], None
    for mask in range(1 << k):
        used, ok = set(), True
        for i in range(k):
            if mask >> i & 1:
                if used & sets[i]:
                    ok = False
                    break
                used |= sets[i]
        if not ok or any(sum(mask >> i & 1 for i in c) > len(c) - 1 for c in cycles):
            continue
        t = 0.0
        for i in range(k):
            if mask >> i & 1:
                t += scores[i]
        if opt is None or t > opt:
            opt, optimal = t, []
        if t == opt:
            optimal.append(mask)
    selected, prefix, inc, exc = [], 0.0, 0, 0
    for v in range(k):
        if prefix == opt:
            break
        cand = inc | (1 << v)
        if any(m & cand == cand and not m & exc for m in optimal):
            inc = cand
            selected.append(v)
            prefix = 0.0
            for w in selected:
                prefix += scores[w]
        else:
            exc |= 1 << v
    return selected, prefix


def contract_solve_cycle(graph, patterns, scores):
    """contract_selection under the reference's cycle elimination loop
    (ilp_solver.cpp:175 solve_with_cycle_elimination)."""
    from paper_1911_11576_b200 import runtime as rt
    sets, cycles = [set(p) for p in patterns], []
    for _ in range(1000):
        sel, tot = contract_selection(scores, sets, cycles)
        c = rt.debug_call("contract", graph=graph, plan=[patterns[i] for i in sel])
        if "cycle" not in c:
            return {"selected": sel, "total": tot}
        cycles.append([sel[k] for k in c["cycle"]["patterns"]])
    raise AssertionError("cycle elimination did not converge")
