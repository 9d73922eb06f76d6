"""Pins of oracle/gate.py and oracle/layer.py: closed forms of silu (P:191,
S:64-69), Eq. 2 zero gating, and central finite differences of the
composed forward for EVERY gradient the backward returns (S:95, S:346,
S:610).  The finite differences only call the forward, so a dropped term,
wrong sign or transposed operand anywhere in the backward fails here."""
import numpy as np
import pytest

from oracle import gate, layer, pkm
from synthetic import gen


def test_silu_closed_forms():
    assert gate.silu(0.0) == 0.0
    assert abs(gate.silu(40.0) - 40.0) < 1e-12
    assert abs(gate.silu(-40.0)) < 1e-12
    assert abs(gate.silu(1.0) - 1.0 / (1.0 + np.exp(-1.0))) < 1e-15
    for x in (-3.0, -0.5, 0.0, 1.0, 2.5):
        h = 1e-6
        fd = (gate.silu(x + h) - gate.silu(x - h)) / (2 * h)
        assert abs(fd - gate.dsilu(x)) < 1e-8


def _inputs(seed, T=3, H=2, S=4, Dk=8, dv=6, D=5, cls=gen.CLS_CONTINUOUS):
    f = lambda tag, shape, sc=1.0: gen.tensor(seed, tag, shape, scale=sc, cls=cls).astype(np.float64)
    return dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)),
                K1=f("K1", (H, S, Dk // 2)), K2=f("K2", (H, S, Dk // 2)),
                V=f("V", (S * S, dv)), W1=f("W1", (D, dv)), W2=f("W2", (dv, D)),
                dout=f("dout", (T, D)))


def test_zero_input_zero_gated_output():
    """x = 0 -> silu(0) = 0 -> output 0."""
    p = _inputs(0)
    out, _ = layer.memory_layer_fwd(np.zeros_like(p["x"]), p["q"], p["K1"], p["K2"],
                                    p["V"], p["W1"], p["W2"], k=2)
    assert np.all(out == 0)


def _loss(p, k, gated, qk_norm=False):
    out, saved = layer.memory_layer_fwd(p["x"], p["q"], p["K1"], p["K2"], p["V"],
                                        p["W1"], p["W2"], k, gated=gated, qk_norm=qk_norm)
    return float((out * p["dout"]).sum()), saved


@pytest.mark.parametrize("gated,qk_norm", [(True, False), (False, False), (True, True)])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_finite_differences_all_gradients(gated, qk_norm, seed):
    """n=8, sqrt(N)=4, k=2: rel. err < 1e-4 for every parameter
    (also with qk-normalisation)."""
    k = 2
    p = _inputs(seed)
    if not gated:   # ungated Memory: out = y, so dout is [T, dv]
        p["dout"] = gen.tensor(seed, "dout", (p["x"].shape[0], p["V"].shape[1])).astype(np.float64)
    _, saved = _loss(p, k, gated, qk_norm)
    g = layer.memory_layer_bwd(p["dout"], p["x"], p["q"], p["K1"], p["K2"], p["V"],
                               p["W1"], p["W2"], saved, gated=gated)
    N, dv = p["V"].shape
    dV_dense = np.zeros((N, dv))
    dV_dense[g["rows"]] = g["dV"]
    analytic = dict(q=g["dq"], K1=g["dK1"], K2=g["dK2"], V=dV_dense)
    if gated:
        analytic.update(x=g["dx"], W1=g["dW1"], W2=g["dW2"])
    h = 1e-6
    for name, ga in analytic.items():
        fd = np.zeros_like(p[name])
        it = np.nditer(p[name], flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            old = p[name][i]
            p[name][i] = old + h
            lp, sp = _loss(p, k, gated, qk_norm)
            p[name][i] = old - h
            lm, sm = _loss(p, k, gated, qk_norm)
            p[name][i] = old
            # the selection must not flip inside the stencil (Q8)
            assert np.array_equal(sp["idx"], saved["idx"]) and np.array_equal(sm["idx"], saved["idx"])
            fd[i] = (lp - lm) / (2 * h)
        denom = max(np.abs(fd).max(), np.abs(ga).max(), 1e-8)
        assert np.abs(fd - ga).max() / denom < 1e-4, name


def test_k1_key_and_query_grads_vanish():
    """k = 1 -> softmax is the constant 1, so dq = dK = 0, and the V
    row gradient is dy of that token."""
    p = _inputs(4)
    out, saved = layer.memory_layer_fwd(p["x"], p["q"], p["K1"], p["K2"], p["V"],
                                        p["W1"], p["W2"], k=1)
    g = layer.memory_layer_bwd(p["dout"], p["x"], p["q"], p["K1"], p["K2"], p["V"],
                               p["W1"], p["W2"], saved)
    assert np.all(g["dq"] == 0) and np.all(g["dK1"] == 0) and np.all(g["dK2"] == 0)
    assert np.all(saved["w"] == 1.0)


def test_two_equal_top_scores_average():
    """two keys with equal scores, k = 2 -> y = average of the rows."""
    S, Dk, dv = 4, 4, 3
    K1 = np.zeros((1, S, 2)); K2 = np.zeros((1, S, 2))
    K1[0, 1] = [1.0, 0.0]; K1[0, 2] = [1.0, 0.0]   # a=1 and a=2 tie
    K2[0, 3] = [0.0, 1.0]
    q = np.array([[[2.0, 0.0, 0.0, 1.0]]])
    V = gen.tensor(1, "V", (S * S, dv)).astype(np.float64)
    idx, score, w = pkm.pkm_lookup(q, K1, K2, 2)
    assert idx[0, 0].tolist() == [1 * S + 3, 2 * S + 3]
    y = layer.memory_layer_fwd(np.zeros((1, 2)), q, K1, K2, V, None, None, 2, gated=False)[0]
    np.testing.assert_allclose(y[0], 0.5 * (V[7] + V[11]), rtol=1e-15)
