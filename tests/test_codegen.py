"""Stitched-kernel generation without a GPU: every plan bench.py and the GPU
tests run generates and compiles (NVRTC, sm_100a) here, with the
composition scheme the design calls for."""
import pytest

from paper_1911_11576_b200 import runtime as rt
from paper_1911_11576_b200 import tuning
from paper_1911_11576_b200 import workloads as W


def compile_only(fused, **kw):
    return rt.Executor(fused, compile_only=True, **kw)


@pytest.mark.parametrize("name", list(W.CONFIGS))
@pytest.mark.parametrize("size", ["small", "full"])
def test_b200_plans_compile(name, size):
    g = W.CONFIGS[name](**(W.SMALL[name] if size == "small" else {}))
    if size == "full":
        fused = tuning.config_plan(name, g)[0]["fused"]  # the bench plan (shipped for bert)
    else:
        fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    ex = compile_only(fused)
    groups = sum(1 for n in fused["nodes"] if n["kind"] == "fused")
    unfused = sum(1 for n in fused["nodes"] if n["kind"] in ("elementwise", "reduce", "dot", "batched_dot"))
    # one kernel per fusion group / kernel op, except unfused broadcasts of
    # constants, which are folded into their consumers as literals
    assert len(ex.info["kernels"]) + ex.info["folded_constant_kernels"] == groups + unfused
    for k in ex.info["kernels"]:
        assert k["block"] % 32 == 0 and k["smem_bytes"] <= 232448


def test_expected_schemes():
    g = W.layernorm()
    ex = compile_only(rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"])
    (k,) = ex.info["kernels"]
    assert k["scheme"].startswith("row_warp") and {"thread", "warp"} <= set(k["composition"])
    g = W.gru()
    ex = compile_only(rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"])
    (k,) = ex.info["kernels"]
    assert "row_cta" in k["scheme"] and "block" in k["composition"] and k["flops"] == 2 * 2 * 4096 * 64 ** 3


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_sectioned_fallback_compiles(name):
    g = W.CONFIGS[name](**W.SMALL[name])
    fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    ex = compile_only(fused, allow_row=False)
    assert all(k["scheme"] in ("sectioned", "flat") for k in ex.info["kernels"])


def test_unfused_baseline_one_kernel_per_op():
    g = W.softmax(**W.SMALL["softmax"])
    ex = compile_only(g, fold_constants=False)  # the bench's unfused baseline
    ops = [n for n in g["nodes"] if n["kind"] in ("elementwise", "reduce", "dot", "batched_dot")]
    assert len(ex.info["kernels"]) == len(ops)
