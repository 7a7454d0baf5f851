"""Host-side checks of the executor's round-2 launch machinery (no GPU:
compile-only executors): the dataflow dependency DAG, split folds, narrow
rows and the L2-discard set, on the bench's BERT plan and on small graphs.
The GPU side (bit-identity of dataflow / serial launch and of discard on /
off) is in tests/test_executor_gpu.py."""
import pytest

from paper_1911_11576_b200 import runtime as rt
from paper_1911_11576_b200 import tuning
from paper_1911_11576_b200 import workloads as W


@pytest.fixture(scope="module")
def bert():
    fused = tuning.config_plan("bert")[0]["fused"]
    ex = rt.Executor(fused, compile_only=True, kernel_options=tuning.kernel_variants("bert"))
    yield fused, ex
    ex.close()


def test_bert_dataflow_dag(bert):
    _, ex = bert
    info = ex.info
    assert info["launch_order"] == "dataflow" and info["concurrent_lanes"] >= 2
    ks = info["kernels"]
    names = [k["name"] for k in ks]
    pos = {n: i for i, n in enumerate(names)}
    # producer of every value (a fold writes only its column reductions, the
    # row kernel the rest; both carry the same argument list)
    folds = {k["name"]: k["fold_of"] for k in ks if k.get("fold_of")}
    assert folds, "no split row groups in the BERT plan"
    for f, row in folds.items():
        assert pos[f] == pos[row] + 1  # launch index right after its row kernel
        assert row in next(k for k in ks if k["name"] == f)["after"]
    writer = {}
    for k in ks:
        if k["name"] in folds:
            continue
        for o in k["outputs"]:
            writer[o] = k["name"]
    for k in ks:
        if k["name"] in folds:
            continue
        for i in k["inputs"]:
            w = writer.get(i)
            if w and w != k["name"]:
                # a value written by a split row kernel may come from its fold
                assert w in k["after"] or any(folds.get(a) == w for a in k["after"]), (k["name"], i, w)
    # after split folds no kernel needs a grid barrier
    assert not any(k["cooperative"] for k in ks)
    # the issue order is a topological order of the DAG
    ipos = {k["name"]: k["issue_pos"] for k in ks}
    assert sorted(ipos.values()) == list(range(len(ks)))
    for k in ks:
        for a in k["after"]:
            assert ipos[a] < ipos[k["name"]], (a, k["name"])


def test_serial_order_has_no_dag(bert):
    fused, _ = bert
    ex = rt.Executor(fused, compile_only=True, kernel_options=tuning.kernel_variants("bert"), concurrent_lanes=1)
    assert ex.info["launch_order"] == "serial" and ex.info["dependency_edges"] == 0
    assert all("after" not in k for k in ex.info["kernels"])
    ex.close()


def test_split_cross_off_restores_grid_barrier(bert):
    fused, on = bert
    off = rt.Executor(fused, compile_only=True, kernel_options=tuning.kernel_variants("bert"), split_cross=False)
    n_fold = sum(1 for k in on.info["kernels"] if k.get("fold_of"))
    n_coop = sum(1 for k in off.info["kernels"] if k["cooperative"])
    assert n_fold == n_coop and n_fold > 0
    assert len(on.info["kernels"]) == len(off.info["kernels"]) + n_fold
    off.close()


def test_narrow_rows_scheme():
    # softmax over 128 keys: a row of 128 elements -> 8 lanes per row
    g = W.softmax(heads=2, seq=128)
    fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    ex = rt.Executor(fused, compile_only=True)
    assert any("nt=8" in k["scheme"] for k in ex.info["kernels"]), [k["scheme"] for k in ex.info["kernels"]]
    wide = rt.Executor(fused, compile_only=True, narrow_rows=False)
    assert not any("nt=8" in k["scheme"] for k in wide.info["kernels"])
    ex.close()
    wide.close()


def test_l2_discard_only_single_reader_intermediates(bert):
    _, ex = bert
    ks = ex.info["kernels"]
    outs = {t["id"] for t in ex.info["outputs"]}
    readers = {}
    for k in ks:
        if k.get("fold_of"):
            continue
        for i in set(k["inputs"]):
            readers[i] = readers.get(i, 0) + 1
    src = ex.sources()
    n = 0
    for k in ks:
        body = src[k["name"]].split('extern "C"')[-1]
        for line in body.splitlines():
            if "discard_l2(" in line:
                n += 1
                vid = line.split("// ")[-1].split(" (dead")[0].strip()
                assert vid not in outs
                assert vid in k["inputs"]
                assert readers.get(vid, 1) == 1, (k["name"], vid, readers.get(vid))
    assert n > 0
    off = rt.Executor(tuning.config_plan("bert")[0]["fused"], compile_only=True,
                      kernel_options=tuning.kernel_variants("bert"), l2_discard=False)
    assert not any("discard_l2(" in s.split('extern "C"')[-1] for s in off.sources().values())
    off.close()
