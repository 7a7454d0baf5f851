"""SPEC known-answer examples and acceptance criteria, run against the
product planner only (no reference needed). Values are the reference
SPEC's [PAPER]/[TRIVIAL]/[DERIVED] examples."""
import json
import os

import pytest

from paper_1911_11576_b200 import runtime as rt

HERE = os.path.dirname(os.path.abspath(__file__))


def golden_graph(name):
    with open(os.path.join(HERE, "golden", "plans.json")) as f:
        for e in json.load(f):
            if e["name"].startswith("fixture:%s@" % name):
                return e["graph"]
    raise KeyError(name)


def p(id, dims):
    return {"id": id, "kind": "parameter", "shape": {"dims": dims, "dtype": "f32"}}


def ew(id, name, ops, dims):
    return {"id": id, "kind": "elementwise", "name": name, "operands": ops, "shape": {"dims": dims, "dtype": "f32"}}


def test_topological_tie_break():
    g = {"nodes": [p("a", [4]), ew("d", "add", ["b", "c"], [4]), ew("c", "exp", ["a"], [4]), ew("b", "exp", ["a"], [4])],
         "outputs": ["d"]}
    assert rt.debug_call("topo", graph=g) == ["a", "b", "c", "d"]


def test_contract_fig3_cycle():
    g = {"nodes": [p("x", [4]), ew("A", "exp", ["x"], [4]), ew("B", "exp", ["A"], [4]), ew("C", "add", ["A", "B"], [4])],
         "outputs": ["C"]}
    r = rt.debug_call("contract", graph=g, plan=[["A", "C"]])
    assert "cycle" in r and r["cycle"]["nodes"] == ["B"]
    r = rt.debug_call("contract", graph=g, plan=[["A", "B"]])
    assert "graph" in r


def test_substitution_chain():
    g = {"nodes": [p("x", [4]), ew("A", "exp", ["x"], [4]), ew("B", "exp", ["A"], [4]), ew("C", "exp", ["B"], [4]),
                   ew("D", "exp", ["C"], [4])], "outputs": ["D"]}
    pats = rt.debug_call("substitution", graph=g, parts=["C"])
    assert [q["nodes"] for q in pats] == [["A", "B"], ["D"]]
    assert rt.debug_call("substitution", graph=g, parts=["A", "B", "C", "D"]) == []


def test_exploratory_chain():
    g = {"nodes": [p("x", [1 << 20]), ew("e1", "exp", ["x"], [1 << 20]), ew("e2", "exp", ["e1"], [1 << 20]),
                   ew("e3", "exp", ["e2"], [1 << 20])], "outputs": ["e3"]}
    pats = rt.debug_call("exploratory", graph=g, seed=["e2"])
    assert sorted(sorted(q["nodes"]) for q in pats) == [["e1", "e2"], ["e1", "e2", "e3"], ["e2", "e3"]]


def test_saved_bytes():
    g = {"nodes": [p("x", [4, 4]), ew("a", "exp", ["x"], [4, 4]), ew("b", "exp", ["a"], [4, 4]),
                   ew("c", "negate", ["a"], [4, 4]), ew("d", "add", ["b", "c"], [4, 4])], "outputs": ["d"]}
    assert rt.debug_call("pattern_info", graph=g, nodes=["a"])["saved_bytes"] == 0
    assert rt.debug_call("pattern_info", graph=g, nodes=["a", "b"])["saved_bytes"] == 64 + 0  # a still read by c
    assert rt.debug_call("pattern_info", graph=g, nodes=["a", "b", "c"])["saved_bytes"] == 192


def test_m_of_v_known():
    # default model table point: 1 MiB -> latency = bytes / bandwidth
    r = rt.debug_call("m_of_v", v=[0, 1 << 20])
    assert r[0][0] == 0.0
    assert r[1][0] == pytest.approx((1 << 20) / r[1][1] * 1e6, rel=1e-12)


def test_score_execution_known():
    r = rt.debug_call("score_execution", nodes=["a", "b", "c"], per_op_us=[5, 5, 5], fused_us=10.0)
    assert r["score"] == 21.0
    r = rt.debug_call("score_execution", nodes=["a", "b", "c"], per_op_us=[5, 5, 5], fused_us=31.0)
    assert r["score"] == 0.0
    r = rt.debug_call("score_execution", nodes=["a", "b", "c"], per_op_us=[5, 5, 5], fused_us=None)
    assert r["score"] == -1.0 and not r["feasible"]


def test_fig1_pipeline():
    """SPEC acceptance 4: Fig 1 fuses into one op (compression 13), add
    reuses dot_1's 94*94*4 = 35,344 shared bytes, alloc/req = 0.5."""
    g = golden_graph("fig1")
    res = rt.plan(g)
    fused = [n for n in res["fused"]["nodes"] if n["kind"] == "fused"]
    assert len(fused) == 1
    rep = res["plan"]["report"]
    assert rep["kernel_compression"] == 13.0
    assert rep["shared_stats"]["max_shd_bytes"] == 35344
    assert rep["shared_stats"]["alloc_over_req"] == 0.5
    body_ops = [n["id"] for n in fused[0]["body"]["nodes"] if n["kind"] not in ("parameter", "tuple")]
    info = rt.debug_call("pattern_info", graph=g, nodes=body_ops)
    alloc = {e["op"]: e for e in info["alloc"]["entries"]}
    assert alloc["add"].get("reused_from") == "dot_1" and info["alloc"]["total"] == 35344


def test_shared_gate_72k():
    """SPEC acceptance 10: a pattern requesting ~72 KB after reuse is
    infeasible at the 48 KiB default, feasible at the B200 227 KiB limit."""
    R = 18432  # 72 KiB of f32 row results
    g = {"nodes": [p("x", [R, 64]),
                   {"id": "r", "kind": "reduce", "operands": ["x"], "reduce_dims": [1], "shape": {"dims": [R], "dtype": "f32"}},
                   {"id": "c", "kind": "reduce", "operands": ["x"], "reduce_dims": [0], "shape": {"dims": [64], "dtype": "f32"}},
                   ew("rb", "broadcast", ["r"], [R, 64]), ew("y", "multiply", ["rb", "x"], [R, 64])],
         "outputs": ["y", "c"]}
    info = rt.debug_call("pattern_info", graph=g, nodes=["r", "rb", "y"])
    assert info["requested"] == R * 4
    assert not info["feasible"]
    info = rt.debug_call("pattern_info", graph=g, nodes=["r", "rb", "y"], shared_limit_bytes=232448)
    assert info["feasible"]


def test_determinism_and_bad_input():
    g = golden_graph("fig1")
    a = rt.plan(g)
    b = rt.plan(g)
    a.pop("timings"), b.pop("timings")
    assert a == b
    with pytest.raises(rt.StitchError) as e:
        rt.plan("{not json")
    assert e.value.code == 1
    bad = {"nodes": [p("x", [4]), ew("y", "add", ["x"], [4])], "outputs": ["y"]}
    with pytest.raises(rt.StitchError) as e:
        rt.plan(bad)
    assert e.value.code == 1
