"""The CPU oracle and its stated tolerance (oracle/executor.py,
oracle/tolerance.py): known answers written independently of the graph
interpreter, and the fp32 error bound holding for an fp32 evaluation while
rejecting real errors."""
import numpy as np
import pytest

from oracle import executor as orc
from oracle import tolerance
from paper_1911_11576_b200 import workloads as W


def test_layernorm_known_answer():
    g = W.layernorm(rows=32, cols=96)
    ins = orc.random_inputs(g, seed=3)
    (y,) = orc.run(g, ins)
    x = ins["x"].astype(np.float64)
    mu = x.mean(1, keepdims=True)
    var = ((x - mu) ** 2).mean(1, keepdims=True)
    ref = (x - mu) / np.sqrt(var + 1e-5) * ins["gamma"] + ins["beta"]
    np.testing.assert_allclose(y, ref, rtol=1e-6, atol=1e-6)


def test_softmax_known_answer():
    g = W.softmax(heads=2, seq=16)
    ins = orc.random_inputs(g, seed=4)
    (p,) = orc.run(g, ins)
    z = ins["x"].astype(np.float64) / 8.0 + ins["mask"]
    z = np.exp(z - z.max(1, keepdims=True))
    np.testing.assert_allclose(p, z / z.sum(1, keepdims=True), rtol=1e-6, atol=1e-7)


def test_gru_known_answer():
    g = W.gru(batch=3, n=8)
    ins = orc.random_inputs(g, seed=5)
    (hn,) = orc.run(g, ins)
    f = {k: v.astype(np.float64) for k, v in ins.items()}
    pre = f["h"] @ f["W"] + f["x"] @ f["U"]
    z = 1 / (1 + np.exp(-pre))
    np.testing.assert_allclose(hn, z * f["h"] + (1 - z) * np.tanh(pre), rtol=1e-5, atol=1e-6)


def test_encoder_dbias_and_broadcast_map():
    g = W.encoder(batch=2, seq=4, hidden=32)
    ins = orc.random_inputs(g, seed=6)
    y, db = orc.run(g, ins)
    np.testing.assert_allclose(db, ins["dy"].astype(np.float64).sum((0, 1)), rtol=1e-6)
    assert orc.broadcast_dim_map([512], [64, 512, 512]) == [2]
    assert orc.broadcast_dim_map([64, 512], [64, 512, 512]) == [0, 2]


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_bound_covers_fp32_evaluation(name):
    g = W.CONFIGS[name](**W.SMALL[name])
    ins = orc.random_inputs(g, seed=7)
    ref, bound = tolerance.reference_with_bound(g, ins)
    got = orc.run(g, ins, dtype=np.float32)
    for a, r, b in zip(got, ref, bound):
        ok, worst = tolerance.check(a, r, b)
        assert ok, worst


def test_bound_rejects_real_errors():
    g = W.layernorm(rows=16, cols=64)
    ins = orc.random_inputs(g, seed=8)
    (r,), (b,) = tolerance.reference_with_bound(g, ins)
    bad = r.copy()
    bad[3, 5] += 1e-3
    assert not tolerance.check(bad, r, b)[0]
    bad = r.copy()
    bad[7] = r[6]  # a wrong row
    assert not tolerance.check(bad, r, b)[0]
