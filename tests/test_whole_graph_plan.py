"""The whole-graph BERT plan (200k candidate patterns, beyond the reference's
exhaustive search) is solved exactly and is the one shipped in
data/plans/bert.json (which bench.py runs)."""
from paper_1911_11576_b200 import runtime as rt
from paper_1911_11576_b200 import tuning
from paper_1911_11576_b200 import workloads as W


def test_bert_plan_exact_and_shipped():
    g = W.bert()
    opts = dict({"shared_limit_bytes": W.B200_SHARED_LIMIT}, **W.PLAN_OPTIONS.get("bert", {}))
    r = rt.plan(g, **opts)
    t = r["timings"]
    assert t["ilp_truncated"] == 0 and t["ilp_lp_gap"] == 0.0
    shipped = tuning.cached_plan("bert", g, opts)
    assert shipped is not None, "data/plans/bert.json is stale: rerun scripts/make_plan_cache.py bert"
    assert shipped["fused"] == r["fused"]
    assert shipped["plan"]["total_score_us"] == r["plan"]["total_score_us"]
    sel = [r["plan"]["patterns"][i] for i in r["plan"]["selected"]]
    assert shipped["plan"]["patterns"]["selected"] == sel
    assert shipped["plan"]["patterns"]["count"] == len(r["plan"]["patterns"])
