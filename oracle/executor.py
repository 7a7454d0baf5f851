"""Test infrastructure (oracle) -- CPU per-op interpreter for graph numerics.

NOT part of the product: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference legs may import this module, and only as the
checker or the timed CPU baseline.

The reference (proj/) plans and emits kernel text but never executes a
graph (SPEC fusion-transform Non-goals), so its op semantics are defined by
the C expressions its emitter writes for each op. This interpreter restates
them op by op, in float64 by default:

  add/subtract/multiply/divide   a+b, a-b, a*b, a/b     emitter.cpp:897-900
  maximum/minimum                fmaxf / fminf          emitter.cpp:901-902
  log/exp/negate/rsqrt           logf/expf/-(x)/rsqrtf  emitter.cpp:903-906
  compare                        (a > b) ? 1 : 0        emitter.cpp:907-911
  select                         (p != 0) ? a : b       emitter.cpp:912-915
  broadcast                      in[coords[map[i]]], map = right-most greedy
                                 subsequence match      graph.cpp:158, emitter.cpp:890-895
  reduce                         sum over reduce_dims   emitter.cpp:808-831
                                 (extension: "name": "max" -> max; the
                                 reference emitter sums every reduce)
  dot                            sum_k lhs[..k..]*rhs[..k..], output dims =
                                 lhs minus cd0 then rhs minus cd1
                                                        emitter.cpp:833-876
  batched_dot                    per batch [M,K] x [K,N] emitter.cpp:850-861
  constant                       the node's "value" (extension; the reference
                                 has no constant data -- its kernels take
                                 constants as pointer arguments)

Pinned: the reference's own emitted kernels (tests/golden/ref_sketches.json,
from oracle/_ref for the six reference fixtures and the SMALL configs, fused
and one-kernel-per-op) are compiled for sm_100a and run on a B200 by
oracle/ref_sketches.py; tests/test_ref_sketches.py checks this interpreter
against their outputs at the stated tolerance. Everything structural (plans,
indexing) is checked against the reference planner through oracle/_ref.
"""

import numpy as np


def broadcast_dim_map(in_dims, out_dims):
    """Right-most greedy subsequence match (reference graph.cpp:158)."""
    m = [-1] * len(in_dims)
    o = len(out_dims) - 1
    for i in range(len(in_dims) - 1, -1, -1):
        while o >= 0 and out_dims[o] != in_dims[i]:
            o -= 1
        if o < 0:
            return None
        m[i] = o
        o -= 1
    return m


def _broadcast(x, out_dims):
    in_dims = list(x.shape)
    if len(in_dims) == 0:
        return np.broadcast_to(x, out_dims)
    m = broadcast_dim_map(in_dims, out_dims)
    if m is None:
        raise ValueError("broadcast input dims are not a subsequence of output dims")
    shape = [1] * len(out_dims)
    for i, d in enumerate(m):
        shape[d] = in_dims[i]
    return np.broadcast_to(x.reshape(shape), out_dims)


def _elementwise(name, args, out_dims, dtype):
    a = args
    if name == "broadcast":
        return _broadcast(a[0], out_dims)
    if name == "add":
        return a[0] + a[1]
    if name == "subtract":
        return a[0] - a[1]
    if name == "multiply":
        return a[0] * a[1]
    if name == "divide":
        with np.errstate(divide="ignore", invalid="ignore"):
            return a[0] / a[1]
    if name == "maximum":
        return np.fmax(a[0], a[1])
    if name == "minimum":
        return np.fmin(a[0], a[1])
    if name == "log":
        with np.errstate(divide="ignore", invalid="ignore"):
            return np.log(a[0])
    if name == "exp":
        with np.errstate(over="ignore"):
            return np.exp(a[0])
    if name == "negate":
        return -a[0]
    if name == "rsqrt":
        with np.errstate(divide="ignore", invalid="ignore"):
            return 1.0 / np.sqrt(a[0])
    if name == "compare":
        return (a[0] > a[1]).astype(dtype)
    if name == "select":
        return np.where(a[0] != 0, a[1], a[2])
    raise ValueError("unknown elementwise op " + name)


def _dot(node, lhs, rhs):
    cd = node.get("contract_dims")
    if cd is None or cd[0] < 0:
        cd = [lhs.ndim - 1, max(0, rhs.ndim - 2)]
    return np.tensordot(lhs, rhs, axes=([cd[0]], [cd[1]]))


def evaluate(graph, inputs, dtype=np.float64, keep=None):
    """Evaluates every node of `graph` (reference JSON format) in dependency
    order. `inputs` maps parameter ids (and constants without a value) to
    arrays. Returns {id: array} for all nodes (tuples map to lists)."""
    nodes = {n["id"]: n for n in graph["nodes"]}
    vals = {}

    def value(nid):
        if nid in vals:
            return vals[nid]
        stack = [nid]
        while stack:
            cur = stack[-1]
            if cur in vals:
                stack.pop()
                continue
            pending = [o for o in nodes[cur].get("operands", []) if o not in vals]
            if pending:
                stack.extend(pending)
                continue
            stack.pop()
            vals[cur] = _eval_node(nodes[cur], vals, inputs, dtype)
        return vals[nid]

    for n in graph["nodes"]:
        value(n["id"])
    return vals


def _eval_node(node, vals, inputs, dtype):
    kind = node["kind"]
    dims = list(node["shape"]["dims"])
    args = [vals[o] for o in node.get("operands", [])]
    if kind == "parameter":
        return np.asarray(inputs[node["id"]], dtype=dtype).reshape(dims)
    if kind == "constant":
        if "value" in node:
            return np.full(dims, node["value"], dtype=dtype)
        return np.asarray(inputs[node["id"]], dtype=dtype).reshape(dims)
    if kind == "elementwise":
        out = _elementwise(node["name"], args, dims, dtype)
        return np.ascontiguousarray(np.asarray(out, dtype=dtype).reshape(dims))
    if kind == "reduce":
        axes = tuple(node["reduce_dims"])
        if node.get("name") == "max":
            return np.max(args[0], axis=axes).reshape(dims)
        return np.sum(args[0], axis=axes).reshape(dims)
    if kind == "dot":
        return _dot(node, args[0], args[1]).reshape(dims)
    if kind == "batched_dot":
        return np.matmul(args[0], args[1]).reshape(dims)
    if kind == "tuple":
        return list(args)
    if kind == "get_element":
        return args[0][node["index"]]
    if kind == "fused":
        body = node["body"]
        params = [n["id"] for n in body["nodes"] if n["kind"] == "parameter"]
        bvals = evaluate(body, dict(zip(params, args)), dtype)
        out = bvals[body["outputs"][0]]
        return out if len(out) > 1 else out[0]
    raise ValueError("unknown op kind " + kind)


def graph_inputs(graph):
    """Parameter ids (and value-less constants) in node order: the executor's
    input order (include/stitch_b200.h stitch_executor_describe)."""
    return [n["id"] for n in graph["nodes"]
            if n["kind"] == "parameter" or (n["kind"] == "constant" and "value" not in n)]


def graph_outputs(graph):
    """Graph outputs flattened through tuples, in order."""
    nodes = {n["id"]: n for n in graph["nodes"]}
    out = []
    for o in graph["outputs"]:
        if nodes[o]["kind"] == "tuple":
            out.extend(nodes[o]["operands"])
        else:
            out.append(o)
    return out


def random_inputs(graph, seed=0, scale=1.0):
    """Seeded fp32 inputs for every graph input (normal, times `scale`)."""
    rng = np.random.default_rng(seed)
    nodes = {n["id"]: n for n in graph["nodes"]}
    return {i: (rng.standard_normal(nodes[i]["shape"]["dims"]) * scale).astype(np.float32)
            for i in graph_inputs(graph)}


def run(graph, inputs, dtype=np.float64):
    """Graph outputs (flattened) as float32 arrays, computed in `dtype`."""
    vals = evaluate(graph, inputs, dtype)
    return [np.asarray(vals[o], dtype=np.float32) for o in graph_outputs(graph)]
