"""Test infrastructure (oracle) -- the stated fp32 tolerance.

NOT part of the product: only tests/, __graft_entry__.smoke() and bench.py's
checker legs import this module.

The stitched kernels compute in fp32; the oracle (oracle/executor.py)
computes in fp64. The acceptance rule (BASELINE.json north_star) is
"within 1e-5 relative or 1e-6 absolute, with the reduction-order tolerance
stated". This module states that tolerance per element:

    |got - ref| <= max(RTOL * |ref|, ATOL) + SAFETY * bound

where `bound` is a first-order forward rounding-error bound of evaluating the
same graph in fp32 (unit roundoff u = 2^-24) in ANY summation order:

    parameter        0 (inputs are exact fp32 values)
    constant         u |c|                  (the literal is rounded to fp32)
    a +- b           ea + eb + u |r|
    a * b            |b| ea + |a| eb + ea eb + u |r|
    a / b            (ea + |r| eb) / (|b| - eb) + u |r|      (inf if |b| <= eb)
    exp(a)           |r| (exp(ea) - 1) + 2u |r|             (expf: <= 2 ulp)
    log(a)           ea / (|a| - ea) + 2u |r|               (logf: <= 2 ulp)
    rsqrt(a)         |r| (1/sqrt(1 - ea/|a|) - 1) + 2u |r|  (rsqrtf: <= 2 ulp)
    negate/broadcast ea (exact)
    max / min        max(ea, eb)
    compare          1 where |a - b| <= ea + eb (the predicate may flip), else 0
    select           e of the chosen branch; |a - b| + ea + eb where the
                     predicate itself is uncertain
    sum over n       sum e_i + (n - 1) u sum |x_i|   <- the reduction-order
                     term: the classic worst case over every association
                     (sequential, shuffle trees, blocked and cross-CTA
                     combines alike)
    max reduce       max e_i (exact)
    |r| + e > FLT_MAX  inf: the fp32 value may overflow, every element that
                     depends on it is uncertified (the check skips it)
    dot (K terms)    |A| eB + eA |B| + K u |A||B|

The fp64 oracle's own error is far below these bounds. SAFETY = 2 covers the
dropped second-order terms.
"""

import numpy as np

from . import executor as orc

U = 2.0 ** -24
RTOL = 1e-5
ATOL = 1e-6
SAFETY = 2.0
FLT_MAX = float(np.finfo(np.float32).max)


def _eval(node, vals, errs, inputs):
    kind = node["kind"]
    dims = list(node["shape"]["dims"])
    ops = node.get("operands", [])
    a = [vals[o] for o in ops]
    e = [errs[o] for o in ops]
    if kind == "parameter":
        v = np.asarray(inputs[node["id"]], dtype=np.float64).reshape(dims)
        return v, np.zeros_like(v)
    if kind == "constant":
        if "value" in node:
            v = np.full(dims, node["value"], dtype=np.float64)
        else:
            v = np.asarray(inputs[node["id"]], dtype=np.float64).reshape(dims)
        return v, U * np.abs(v)
    if kind == "tuple":
        return list(a), list(e)
    if kind == "elementwise":
        name = node["name"]
        if name == "broadcast":
            return (np.ascontiguousarray(orc._broadcast(a[0], dims)),
                    np.ascontiguousarray(orc._broadcast(e[0], dims)))
        with np.errstate(all="ignore"):
            r = np.asarray(orc._elementwise(name, a, dims, np.float64), dtype=np.float64).reshape(dims)
            ar = np.abs(r)
            if name in ("add", "subtract"):
                err = e[0] + e[1] + U * ar
            elif name == "multiply":
                err = np.abs(a[1]) * e[0] + np.abs(a[0]) * e[1] + e[0] * e[1] + U * ar
            elif name == "divide":
                den = np.abs(a[1]) - e[1]
                err = np.where(den > 0, (e[0] + ar * e[1]) / np.where(den > 0, den, 1.0), np.inf) + U * ar
            elif name == "exp":
                err = ar * np.expm1(e[0]) + 2 * U * ar
            elif name == "log":
                den = np.abs(a[0]) - e[0]
                err = np.where(den > 0, e[0] / np.where(den > 0, den, 1.0), np.inf) + 2 * U * ar
            elif name == "rsqrt":
                q = e[0] / np.abs(a[0])
                err = np.where(q < 1, ar * (1.0 / np.sqrt(np.maximum(1 - q, 1e-300)) - 1.0), np.inf) + 2 * U * ar
            elif name == "negate":
                err = e[0].copy()
            elif name in ("maximum", "minimum"):
                err = np.maximum(e[0], e[1])
            elif name == "compare":
                err = (np.abs(a[0] - a[1]) <= e[0] + e[1]).astype(np.float64)
            elif name == "select":
                unsure = np.abs(a[0]) <= e[0]
                chosen = np.where(a[0] != 0, e[1], e[2])
                err = np.where(unsure, np.abs(a[1] - a[2]) + e[1] + e[2], chosen)
            else:
                raise ValueError("unknown elementwise op " + name)
        return r, err
    if kind == "reduce":
        axes = tuple(node["reduce_dims"])
        if node.get("name") == "max":
            return np.max(a[0], axis=axes).reshape(dims), np.max(e[0], axis=axes).reshape(dims)
        n = int(np.prod([a[0].shape[d] for d in axes]))
        v = np.sum(a[0], axis=axes).reshape(dims)
        err = (np.sum(e[0], axis=axes) + (n - 1) * U * np.sum(np.abs(a[0]), axis=axes)).reshape(dims)
        return v, err
    if kind in ("dot", "batched_dot"):
        A, B, eA, eB = a[0], a[1], e[0], e[1]
        if kind == "dot":
            cd = node.get("contract_dims")
            if cd is None or cd[0] < 0:
                cd = [A.ndim - 1, max(0, B.ndim - 2)]
            K = A.shape[cd[0]]
            mm = lambda x, y: np.tensordot(x, y, axes=([cd[0]], [cd[1]]))
        else:
            K = A.shape[-1]
            mm = np.matmul
        v = mm(A, B).reshape(dims)
        err = (mm(np.abs(A), eB) + mm(eA, np.abs(B)) + K * U * mm(np.abs(A), np.abs(B))).reshape(dims)
        return v, err
    if kind == "get_element":
        return a[0][node["index"]], e[0][node["index"]]
    if kind == "fused":
        body = node["body"]
        params = [n["id"] for n in body["nodes"] if n["kind"] == "parameter"]
        bv, be = _evaluate(body, dict(zip(params, a)), dict(zip(params, e)))
        out = body["outputs"][0]
        return bv[out], be[out]
    raise ValueError("unknown op kind " + kind)


def _evaluate(graph, inputs, input_errs=None):
    vals, errs = {}, {}
    nodes = {n["id"]: n for n in graph["nodes"]}
    order = []
    seen = set()

    def visit(nid):
        stack = [(nid, False)]
        while stack:
            cur, done = stack.pop()
            if done:
                order.append(cur)
                continue
            if cur in seen:
                continue
            seen.add(cur)
            stack.append((cur, True))
            for o in nodes[cur].get("operands", []):
                if o not in seen:
                    stack.append((o, False))

    for n in graph["nodes"]:
        visit(n["id"])
    # free every value after its last consumer (whole-graph configs hold
    # thousands of intermediates); graph outputs and tuple members stay
    keep = set(graph["outputs"])
    for o in graph["outputs"]:
        if nodes[o]["kind"] == "tuple":
            keep.update(nodes[o]["operands"])
    uses = {}
    for n in graph["nodes"]:
        for o in n.get("operands", []):
            uses[o] = uses.get(o, 0) + 1
    for nid in order:
        node = nodes[nid]
        if input_errs is not None and node["kind"] == "parameter":
            vals[nid] = np.asarray(inputs[nid], dtype=np.float64)
            errs[nid] = np.asarray(input_errs[nid], dtype=np.float64)
        else:
            vals[nid], errs[nid] = _eval(node, vals, errs, inputs)
            if node["kind"] not in ("tuple", "fused", "parameter"):
                # a value that may exceed the fp32 range overflows to inf in
                # the kernel (and to NaN downstream): uncertified from here on
                with np.errstate(all="ignore"):
                    e = np.nan_to_num(errs[nid], nan=np.inf, posinf=np.inf)
                    errs[nid] = np.where(np.abs(vals[nid]) + e > FLT_MAX, np.inf, e)
        if node["kind"] not in ("tuple", "fused"):
            for o in node.get("operands", []):
                uses[o] -= 1
                if uses[o] == 0 and o not in keep and nodes[o]["kind"] != "tuple":
                    vals.pop(o, None)
                    errs.pop(o, None)
    return vals, errs


def reference_with_bound(graph, inputs):
    """(outputs, bounds): the fp64 oracle outputs of `graph` (flattened
    through tuples, executor output order) and the fp32 forward error bound
    of each."""
    vals, errs = _evaluate(graph, inputs)
    outs = orc.graph_outputs(graph)
    return [vals[o] for o in outs], [errs[o] for o in outs]


def check(got, ref, bound):
    """(ok, worst): worst = max |got - ref| / tol over elements (<= 1 passes).
    NaN matches NaN; infinities must match exactly."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if got.shape != ref.shape:
        got = got.reshape(ref.shape)
    # A NaN bound (inf * 0 in a deep chain) is no bound at all: treat it as
    # infinite, i.e. the element is uncertified rather than failed. Deep
    # whole-graph outputs (12 residual + LayerNorm layers) exceed first-order
    # worst-case analysis; tests check those against the unfused GPU graph.
    bound = np.nan_to_num(np.asarray(bound, dtype=np.float64), nan=np.inf, posinf=np.inf)
    tol = np.maximum(RTOL * np.abs(ref), ATOL) + SAFETY * bound
    both_nan = np.isnan(got) & np.isnan(ref)
    same_inf = np.isinf(ref) & (got == ref)
    with np.errstate(invalid="ignore"):
        ratio = np.abs(got - ref) / tol
    ratio = np.where(both_nan | same_inf | np.isinf(tol), 0.0, ratio)
    ratio = np.where(np.isnan(ratio), np.inf, ratio)
    worst = float(ratio.max()) if ratio.size else 0.0
    return worst <= 1.0, worst


def anchored_graph(graph, anchors):
    """`graph` with every anchor value's CONSUMERS reading a parameter
    "<id>@anchor" instead of the anchor itself; the anchor keeps its own
    definition (it is still checked, from its own anchored operands)."""
    nodes = []
    for n in graph["nodes"]:
        m = dict(n)
        if "operands" in n:
            m["operands"] = [o + "@anchor" if o in anchors else o for o in n["operands"]]
        nodes.append(m)
    shapes = {n["id"]: n["shape"] for n in graph["nodes"]}
    extra = [{"id": a + "@anchor", "kind": "parameter", "shape": shapes[a]} for a in sorted(anchors)]
    return {"nodes": extra + nodes, "outputs": list(graph["outputs"])}


def anchored_reference_with_bound(graph, inputs, got):
    """Step-wise certification for deep graphs (12-layer BERT): every graph
    output that other nodes consume is an anchor; its consumers are
    evaluated from the checked executor's value of it (`got[id]`, fp32), so
    each output's fp64 reference and first-order bound cover only the ops
    since the nearest anchors -- one layer, forward or backward -- instead of
    the whole chain, whose worst-case bound is infinite after 12 LayerNorm
    layers. Anchors are themselves outputs and are checked the same way from
    their own anchors, so every output is certified against the ops between
    two checked values. Returns (outputs, bounds) like reference_with_bound."""
    outs = orc.graph_outputs(graph)
    consumed = {o for n in graph["nodes"] for o in n.get("operands", [])}
    anchors = {o for o in outs if o in consumed}
    g2 = anchored_graph(graph, anchors)
    ins2 = dict(inputs)
    for a in anchors:
        ins2[a + "@anchor"] = np.asarray(got[a], dtype=np.float32)
    return reference_with_bound(g2, ins2)
