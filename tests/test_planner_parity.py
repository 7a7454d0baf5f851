"""Fusion-plan parity: the product planner (libstitch_b200.so, C ABI
stitch_debug_call / stitch_plan_graph) against the REFERENCE planner compiled
from its own sources (oracle/_ref, reference proj/src/*.cpp). Every stage is
compared on identical arguments, bit for bit (scores as IEEE doubles).

Reference functions exercised (file:line in /root/reference/proj/src):
  topological_sort graph.cpp, contract_plan graph.cpp, substitution_fusion /
  multi_step_patterns / exploratory_fusion / select_seeds pattern_gen.cpp,
  saved_bytes / m_of_v / score_model_based / shared_feasible cost_model.cpp,
  canonical_shared_requests / shared_planning / PostDominance emitter.cpp,
  solve / solve_with_cycle_elimination ilp_solver.cpp, apply_plan
  transform.cpp, run_plan pipeline.cpp.
"""
import json
import random

import pytest

from conftest import strip_plan
from helpers import contract_solve_cycle, random_dag
from paper_1911_11576_b200 import runtime as rt
from paper_1911_11576_b200 import workloads as W

FIXTURES = ["fig1", "thread", "warp", "block", "packing", "all_partition"]


def fixture_graph(name):
    with open("/root/reference/proj/fixtures/%s.json" % name) as f:
        return json.load(f)


def both(ref, fn, **args):
    return rt.debug_call(fn, **args), ref.call(fn, **args)


@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("lim", [W.REFERENCE_SHARED_LIMIT, W.B200_SHARED_LIMIT])
def test_fixture_plans(ref, name, lim):
    g = fixture_graph(name)
    a, b = both(ref, "plan", graph=g, shared_limit_bytes=lim)
    assert strip_plan(a) == strip_plan(b)


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_stages(ref, name):
    g = fixture_graph(name)
    for fn in ("topo", "seeds", "multi_step", "generate_patterns"):
        a, b = both(ref, fn, graph=g)
        assert a == b, fn
    pats = rt.debug_call("generate_patterns", graph=g)
    for p in pats:
        a, b = both(ref, "pattern_info", graph=g, nodes=p["nodes"])
        assert a == b, p["nodes"]
        a, b = both(ref, "postdom", graph=g, nodes=p["nodes"])
        assert sorted(map(tuple, a)) == sorted(map(tuple, b))


@pytest.mark.parametrize("name", list(W.CONFIGS))
@pytest.mark.parametrize("lim", [W.REFERENCE_SHARED_LIMIT, W.B200_SHARED_LIMIT])
def test_workload_plans_small(ref, name, lim):
    g = W.CONFIGS[name](**W.SMALL[name])
    a, b = both(ref, "plan", graph=g, shared_limit_bytes=lim)
    assert strip_plan(a) == strip_plan(b)


@pytest.mark.parametrize("seed", range(40))
def test_random_dag_plans(ref, seed):
    g = random_dag(seed, n_ops=6 + seed % 9, dims=(64 + 64 * (seed % 5), 256 * (1 + seed % 4)))
    for fn in ("topo", "multi_step", "generate_patterns"):
        a, b = both(ref, fn, graph=g)
        assert a == b, fn
    a, b = both(ref, "plan", graph=g, shared_limit_bytes=[W.REFERENCE_SHARED_LIMIT, W.B200_SHARED_LIMIT][seed % 2])
    assert strip_plan(a) == strip_plan(b)


@pytest.mark.parametrize("seed", range(30))
def test_random_substitution_and_contract(ref, seed):
    rng = random.Random(seed)
    g = random_dag(seed, n_ops=10)
    ids = [n["id"] for n in g["nodes"] if n["kind"] != "parameter"]
    parts = rng.sample(ids, rng.randint(0, len(ids)))
    a, b = both(ref, "substitution", graph=g, parts=parts)
    assert a == b
    # random disjoint plan for contraction
    pool = ids[:]
    rng.shuffle(pool)
    plan = []
    while pool:
        k = rng.randint(1, 4)
        plan.append(pool[:k])
        pool = pool[k:]
    a, b = both(ref, "contract", graph=g, plan=plan)
    assert a == b


@pytest.mark.parametrize("seed", range(200))
def test_ilp_solve_random(ref, seed):
    """SPEC acceptance 1: random instances (k <= 12), exact optimum equal to
    the reference and to exhaustive enumeration."""
    rng = random.Random(seed)
    k = rng.randint(1, 12)
    scores = [round(rng.uniform(0, 100), rng.choice([0, 1, 3])) for _ in range(k)]
    pairs = [[u, v] for u in range(k) for v in range(u + 1, k) if rng.random() < 0.3]
    cycles = [sorted(rng.sample(range(k), rng.randint(1, min(3, k)))) for _ in range(rng.randint(0, 2))]
    args = dict(num_vars=k, scores=scores, pairs=pairs, cycles=cycles)
    a, b = both(ref, "solve", **args)
    assert a == b
    best = 0.0
    for mask in range(1 << k):
        sel = [i for i in range(k) if mask >> i & 1]
        if any(mask >> u & 1 and mask >> v & 1 for u, v in pairs):
            continue
        if any(sum(mask >> i & 1 for i in c) > len(c) - 1 for c in cycles):
            continue
        tot = 0.0
        for i in sel:
            tot += scores[i]
        best = max(best, tot)
    assert a["total"] == best


@pytest.mark.parametrize("seed", range(40))
def test_cycle_elimination_random(ref, seed):
    """SPEC acceptance 2: adversarial overlapping patterns on random DAGs;
    same plan as the reference and an acyclic contraction."""
    rng = random.Random(1000 + seed)
    g = random_dag(seed, n_ops=8 + seed % 8)
    ids = [n["id"] for n in g["nodes"] if n["kind"] != "parameter"]
    pats = [sorted(rng.sample(ids, rng.randint(1, min(5, len(ids))))) for _ in range(rng.randint(2, 9))]
    scores = [float(rng.randint(1, 50)) for _ in pats]
    a, b = both(ref, "solve_cycle", graph=g, patterns=pats, scores=scores)
    assert a == b
    chosen = [pats[i] for i in a["selected"]]
    assert "cycle" not in rt.debug_call("contract", graph=g, plan=chosen)


@pytest.mark.parametrize("seed", range(80))
def test_cycle_elimination_degenerate(ref, seed):
    """Tie-heavy selection instances (the shape of the whole-graph BERT
    instance): pattern scores are sums of per-op weights, so every way of
    covering the same ops is a tie in real arithmetic and the LP relaxation
    has many zero-reduced-cost columns; only the ascending-order double sums
    separate the ties. Exercises the rounding window, reduced-cost fixing
    and the split into independent pieces against the reference's
    exhaustive search and lexicographic extraction."""
    rng = random.Random(5000 + seed)
    g = random_dag(seed, n_ops=8 + seed % 7)
    ids = [n["id"] for n in g["nodes"] if n["kind"] != "parameter"]
    w = {i: rng.choice([0.1, 0.2, 0.3, 0.7, 1.1, 1e-3, 3.3]) * rng.choice([1, 10, 1e4]) for i in ids}
    pats = []
    for _ in range(rng.randint(4, 14)):
        p = sorted(rng.sample(ids, rng.randint(1, min(4, len(ids)))))
        if p not in pats:
            pats.append(p)
    scores = []
    for p in pats:
        t = 0.0
        for i in (p if rng.random() < 0.5 else reversed(p)):
            t += w[i]
        scores.append(t if rng.random() < 0.9 else 0.0)
    a, b = both(ref, "solve_cycle", graph=g, patterns=pats, scores=scores)
    want = contract_solve_cycle(g, pats, scores)
    assert a == want
    if seed in REFERENCE_ROUNDING_DEFECTS:
        # the reference's own search misses its optimum here (below)
        assert b != want and b["total"] < want["total"]
    else:
        assert a == b
    chosen = [pats[i] for i in a["selected"]]
    assert "cycle" not in rt.debug_call("contract", graph=g, plan=chosen)


# Instances of test_cycle_elimination_degenerate where the reference violates
# its own contract: ValueSearch::descend (ilp_solver.cpp:127) prunes with
# canonical_total() + remaining <= best_, `remaining` being a running double
# difference; on near-tie instances its rounding lands the bound just under
# the canonical optimum, a fixed-prefix probe of the extraction
# (ilp_solver.cpp:160) then never reproduces `optimum` exactly, and the
# reference returns a non-optimal selection (seed 39: the empty one, total
# 0.0, where 11.2 is feasible). This solver follows the contract there
# (brute force: tests/helpers.py contract_selection); 1 of 200 seeds checked.
REFERENCE_ROUNDING_DEFECTS = {39}


@pytest.mark.parametrize("seed", range(20))
def test_shared_planning_random(ref, seed):
    """SPEC acceptance 5 (safety) + parity of the dominance-tree reuse."""
    rng = random.Random(seed)
    g = random_dag(seed, n_ops=10)
    ids = [n["id"] for n in g["nodes"] if n["kind"] != "parameter"]
    nodes = sorted(rng.sample(ids, rng.randint(2, len(ids))))
    reqs = [{"op": i, "bytes": rng.choice([256, 1024, 4096])} for i in nodes if rng.random() < 0.5]
    a, b = both(ref, "shared_planning", graph=g, nodes=nodes, requests=reqs)
    assert a == b
    assert a["total"] <= sum(r["bytes"] for r in reqs)


def test_m_of_v_and_scores(ref):
    vs = [0, 1, 1000, 1 << 20, 3 << 20, 1 << 30, 1 << 40]
    a, b = both(ref, "m_of_v", v=vs)
    assert a == b
    g = fixture_graph("fig1")
    for per, fused in (([5, 5, 5], 10.0), ([1.0, 2.5], None), ([3, 3, 3], 25.0)):
        nodes = ["dot_1", "multiply_1", "exp_1"][: len(per)]
        a, b = both(ref, "score_execution", graph=g, nodes=nodes, per_op_us=per, fused_us=fused)
        assert a == b


@pytest.mark.parametrize("name", ["layernorm", "softmax", "gru"])
def test_execution_based_plans(ref, name):
    """Execution-based scoring (paper §4.3) from the shipped B200 kernel-time
    table: the reference planner with the same CSV evaluator selects the same
    fusion groups. (encoder: tests/golden/plans_exec.json, the reference
    takes minutes.)"""
    from paper_1911_11576_b200 import tuning
    g = W.CONFIGS[name]()
    csv = tuning.load(name)
    a, b = both(ref, "plan", graph=g, mode="execution", kernel_times_csv=csv)
    assert strip_plan(a) == strip_plan(b)
