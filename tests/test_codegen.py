"""Stitched-kernel generation without a GPU: every plan bench.py and the GPU
tests run generates and compiles (NVRTC, sm_100a) here, with the
composition scheme the design calls for."""
import pytest

from paper_1911_11576_b200 import runtime as rt
from paper_1911_11576_b200 import tuning
from paper_1911_11576_b200 import workloads as W

from helpers import _node, chunk_chain_graph


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
    # constants (folded into their consumers as literals) and of small
    # tensors (sunk into their consumers' bodies); a row group with column
    # reductions adds its fold kernel (split_cross)
    folds = [k for k in ex.info["kernels"] if k.get("fold_of")]
    assert all(k["scheme"].startswith("fold(") for k in folds)
    assert (len(ex.info["kernels"]) - len(folds) + ex.info["folded_constant_kernels"] + ex.info["sunk_broadcast_kernels"]
            == groups + unfused)
    for k in ex.info["kernels"]:
        assert k["block"] % 32 == 0 and k["smem_bytes"] <= 232448


def test_expected_schemes():
    g = W.layernorm()
    ex = compile_only(rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"])
    (k,) = ex.info["kernels"]
    assert k["scheme"].startswith("row_warp") and {"thread", "warp"} <= set(k["composition"])
    g = W.gru()
    fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    (k,) = compile_only(fused).info["kernels"]
    # the warp-specialised tcgen05 scheme by default, the FFMA ROW scheme without it
    assert k["scheme"].startswith("gws") and "tensor" in k["composition"] and k["flops"] == 2 * 2 * 4096 * 64 ** 3
    assert k["block"] == 576 and k["smem_bytes"] == 230536
    (k,) = compile_only(fused, gws=False).info["kernels"]
    assert "row_cta" in k["scheme"] and "block" in k["composition"] and k["flops"] == 2 * 2 * 4096 * 64 ** 3


def test_gws_kernel_source_shape():
    """The generated gws kernel: four tensor maps by value, the device
    template with the A0 tile staged for the tail (z * h), branch-free
    power-of-two divides, and the tensor-map parameters the runtime encodes."""
    import os
    import tempfile
    g = W.gru(batch=300)
    fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    d = tempfile.mkdtemp()
    os.environ["STITCH_DUMP_DIR"] = d
    try:
        compile_only(fused)
    finally:
        del os.environ["STITCH_DUMP_DIR"]
    src = open(os.path.join(d, "fusion_0.cu")).read()
    assert src.count("__grid_constant__ stitch_dev::gws::TmaDesc") == 4
    assert "stitch_dev::gws::run<1>(&tm0, &tm1, &tm2, &tm3, 0, 300LL, smem, tail)" in src
    assert "stitch_dev::rcp_nr(" in src and " / " not in src.split("struct Tail")[1].split("static_assert")[0]


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_sectioned_fallback_compiles(name):
    g = W.CONFIGS[name](**W.SMALL[name])
    fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    ex = compile_only(fused, allow_row=False)
    assert all(k["scheme"] in ("sectioned", "flat") for k in ex.info["kernels"])


def test_unfused_baseline_one_kernel_per_op():
    g = W.softmax(**W.SMALL["softmax"])
    ex = compile_only(g, fold_constants=False, sink_broadcasts=False)  # the bench's unfused baseline
    ops = [n for n in g["nodes"] if n["kind"] in ("elementwise", "reduce", "dot", "batched_dot")]
    assert len(ex.info["kernels"]) == len(ops)


def test_chunked_segment_buffers_do_not_alias():
    """every buffer a chunked segment touches is live across the
    whole segment (each chunk runs all of its kernels), so `y` -- written by
    the segment's last kernel, read after it -- may not share memory with
    the chunk rings of `a` and `b`: 4 MiB + 2 rings of 2 x 2 MiB."""
    ex = compile_only(chunk_chain_graph(), chunking=True, chunk_fill=False)
    assert ex.info["schedule"][0]["chunks"] == 2 and len(ex.info["schedule"][0]["kernels"]) == 3
    assert ex.info["arena_bytes"] >= 12 * 2 ** 20


def test_colred_output_feeding_post_op_compiles():
    """a cross-row reduce that is a graph output AND feeds a
    post-reduction op of the same group is read back from its output."""
    R, C = 256, 64
    g = {"nodes": [_node("dy", "parameter", dims=(R, C)), _node("x", "parameter", dims=(R, C)),
                   _node("p", "elementwise", ["dy", "x"], "multiply", dims=(R, C)),
                   _node("rs", "reduce", ["p"], dims=(R,), reduce_dims=[1]),
                   _node("db", "reduce", ["dy"], dims=(C,), reduce_dims=[0]),
                   _node("q", "elementwise", ["db", "db"], "multiply", dims=(C,)),
                   {"id": "t", "kind": "tuple", "operands": ["rs", "db", "q"], "shape": {"dims": [C], "dtype": "f32"}}],
         "outputs": ["t"]}
    fused = rt.plan(g)["fused"]
    assert sum(n["kind"] == "fused" for n in fused["nodes"]) == 1
    compile_only(fused)


def test_broadcast_sinking():
    """Unfused broadcasts of small tensors are not materialised: in the
    per-op BERT graph the bias / LayerNorm gamma broadcasts move into their
    consumers' bodies (fewer kernels, fewer bytes), and a graph output
    broadcast still gets its kernel. (The exact whole-graph plan fuses every
    broadcast into a group; the round-1 truncated plan left 12 unfused.)"""
    f = W.bert(**W.SMALL["bert"])
    on = compile_only(f).info
    off = compile_only(f, sink_broadcasts=False).info
    assert on["sunk_broadcast_kernels"] >= 10
    assert len(on["kernels"]) == len(off["kernels"]) - on["sunk_broadcast_kernels"]
    assert on["algo_bytes"] < off["algo_bytes"]
    R, C = 256, 64
    g = {"nodes": [_node("x", "parameter", dims=(R, C)), _node("gam", "parameter", dims=(C,)),
                   _node("gb", "elementwise", ["gam"], "broadcast", dims=(R, C)),
                   _node("y", "elementwise", ["x", "gb"], "multiply", dims=(R, C)),
                   _node("z", "elementwise", ["gb", "x"], "add", dims=(R, C)),
                   {"id": "t", "kind": "tuple", "operands": ["y", "z"], "shape": {"dims": [R, C], "dtype": "f32"}}],
         "outputs": ["t"]}
    info = compile_only(g).info
    assert info["sunk_broadcast_kernels"] == 1 and len(info["kernels"]) == 2
    g["nodes"][-1]["operands"] = ["y", "z", "gb"]
    info = compile_only(g).info
    assert info["sunk_broadcast_kernels"] == 0 and len(info["kernels"]) == 3


def test_fig1_block_composition():
    """Paper Fig. 1 (the reference's fig1 fixture, one fused group of two
    batched dots, two reductions over different index spaces and elementwise
    ops) runs as BLOCK composition: one CTA per leading index, no grid
    barrier, shared memory exactly the planner's Alg. 4 alloc map (dot_1's
    35,344-byte block reused by add: alloc / requested = 0.5), the second dot
    computed inside its consumer's section."""
    import json
    import os
    fx = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_sketches.json")
    g = next(e for e in json.load(open(fx)) if e["name"] == "fixture:fig1")["graph"]
    for lim in (W.REFERENCE_SHARED_LIMIT, W.B200_SHARED_LIMIT):
        fused = rt.plan(g, shared_limit_bytes=lim)["fused"]
        info = rt.debug_call("pattern_info", graph=g, nodes=[n["id"] for n in g["nodes"] if n["kind"] not in ("parameter", "tuple")])
        assert info["alloc"]["total"] == 35344 and info["requested"] == 2 * 35344
        (k,) = compile_only(fused).info["kernels"]
        assert k["scheme"] == "block(G=1,smem=35344)" and not k["cooperative"]
        assert k["smem_bytes"] - 16 == info["alloc"]["total"]
        assert "block" in k["composition"]


def test_block_scheme_off_falls_back_to_sectioned():
    import json
    import os
    fx = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_sketches.json")
    g = next(e for e in json.load(open(fx)) if e["name"] == "fixture:fig1")["graph"]
    fused = rt.plan(g)["fused"]
    (k,) = compile_only(fused, block_compose=False).info["kernels"]
    assert k["scheme"] == "sectioned" and k["cooperative"]


@pytest.mark.parametrize("seed", range(0, 64, 3))
def test_random_dag_kernels_compile(seed):
    """Every kernel of seeded random DAGs compiles under the default and the
    non-default codegen paths (cluster COLRED grids a multiple of the
    cluster, BLOCK / ROW / COLRED / FLAT)."""
    from helpers import random_dag
    R = [3, 64, 100, 257, 1024, 1, 2, 4096][seed % 8]
    C = [4, 33, 256, 768, 1000, 1, 2, 2048][(seed // 8) % 8]
    g = random_dag(seed, n_ops=6 + seed % 10, dims=(R, C))
    fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    for opts in ({}, dict(row_prefetch_warp=True, colred_cols=128, tma_early=True, cross_smem=False,
                          colred_cp_async=False), dict(colred_cluster=8), dict(colred_cluster=0)):
        for gg in (fused, g):
            for k in compile_only(gg, **opts).info["kernels"]:
                assert k["block"] % 32 == 0


def test_gemm_scheme_selection():
    """A kernel that is one unfused dot / batched dot takes the tiled GEMM
    scheme (reference fixture all_partition: two 512^3 dots the planner
    leaves unfused); a dot fused with other ops does not."""
    nodes = [_node(p, "parameter", dims=(512, 512)) for p in ("p0", "p1", "p2")]
    nodes += [_node("dot_a", "dot", ["p0", "p1"], dims=(512, 512), contract_dims=[1, 0]),
              _node("dot_b", "dot", ["dot_a", "p2"], dims=(512, 512), contract_dims=[1, 0])]
    g = {"nodes": nodes, "outputs": ["dot_b"]}
    ex = compile_only(rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"])
    assert [k["scheme"] for k in ex.info["kernels"]] == ["gemm(1x512x512x512)"] * 2
    src = ex.sources()
    assert "stitch_dev::gemm::run<512LL, 512LL, 512LL, 1LL, 512LL, 1LL, 0LL, 512LL, 1LL, 0LL>" in src["dot_a"]
    ex = compile_only(g, gemm=False)
    assert all(not k["scheme"].startswith("gemm") for k in ex.info["kernels"])
    # transposed operands: strides follow the contraction dims
    g2 = {"nodes": [_node("a", "parameter", dims=(77, 300)), _node("b", "parameter", dims=(130, 77)),
                    _node("c", "dot", ["a", "b"], dims=(300, 130), contract_dims=[0, 1])], "outputs": ["c"]}
    ex = compile_only(g2)
    assert "gemm::run<300LL, 130LL, 77LL, 1LL, 1LL, 300LL, 0LL, 1LL, 77LL, 0LL>" in ex.sources()["c"]
    # fused with an elementwise consumer: not the GEMM scheme
    g3 = {"nodes": [_node("a", "parameter", dims=(64, 64)), _node("b", "parameter", dims=(64, 64)),
                    _node("c", "dot", ["a", "b"], dims=(64, 64)), _node("d", "elementwise", ["c"], "exp", dims=(64, 64))],
          "outputs": ["d"]}
    fused = rt.debug_call("apply_plan", graph=g3, patterns=[["c", "d"]], selected=[0])["graph"]
    ex = compile_only(fused)
    assert not any(k["scheme"].startswith("gemm") for k in ex.info["kernels"])
