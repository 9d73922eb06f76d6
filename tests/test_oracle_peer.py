"""Pins of oracle/peer.py (PEER-style rank-1 experts, SURVEY.md §8(f) f4;
PAPER.md P:139; reading Q21 in DESIGN.md).

* k = 1 closed form: one expert per head with weight 1, y = sum_h silu(U[i_h].x) V[i_h];
* the dense rank-1-matrix formulation: y = sum_j w_j (V[i_j] U[i_j]^T-free form)
  written as an explicit loop over experts with a materialised rank-1 matrix
  M_j = V[i_j] U[i_j]^T applied through the nonlinearity (a different computation);
* x = 0 -> y = 0 (silu(0) = 0); U = 0 -> y = 0;
* every gradient (x, q, K1, K2, U, V) against central finite differences.
"""
import numpy as np
import pytest

from oracle import peer, gate
from synthetic import gen


def _inputs(seed, T=3, H=2, S=4, Dk=8, D=6):
    f = lambda tag, shape: gen.tensor(seed, tag, shape).astype(np.float64)
    return dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)),
                K1=f("K1", (H, S, Dk // 2)), K2=f("K2", (H, S, Dk // 2)),
                U=f("W1", (S * S, D)), V=f("V", (S * S, D)), dy=f("dout", (T, D)))


def test_k1_closed_form():
    p = _inputs(0)
    y, s = peer.peer_fwd(p["x"], p["q"], p["K1"], p["K2"], p["U"], p["V"], k=1)
    assert np.all(s["w"] == 1.0)
    T, H = p["q"].shape[:2]
    for t in range(T):
        ref = np.zeros(p["x"].shape[1])
        for h in range(H):
            i = s["idx"][t, h, 0]
            ref += gate.silu(p["U"][i] @ p["x"][t]) * p["V"][i]
        np.testing.assert_allclose(y[t], ref, rtol=1e-13, atol=1e-15)


def test_rank1_matrix_formulation():
    """Each selected expert is the rank-1 matrix V[i] U[i]^T behind a silu on
    its rank-1 activation: y_t = sum_j w_j * silu(<u_j, x_t>) v_j computed as
    M_j x_t = v_j (u_j . x_t) -> scaled by silu(s)/s (s != 0)."""
    p = _inputs(1)
    k = 3
    y, s = peer.peer_fwd(p["x"], p["q"], p["K1"], p["K2"], p["U"], p["V"], k=k)
    T, H = p["q"].shape[:2]
    for t in range(T):
        ref = np.zeros(p["x"].shape[1])
        for h in range(H):
            for j in range(k):
                i = s["idx"][t, h, j]
                M = np.outer(p["V"][i], p["U"][i])         # the rank-1 expert matrix
                act = p["U"][i] @ p["x"][t]
                ref += s["w"][t, h, j] * (M @ p["x"][t]) * (gate.silu(act) / act)
        np.testing.assert_allclose(y[t], ref, rtol=1e-12, atol=1e-14)


def test_zero_input_or_zero_keys_give_zero():
    p = _inputs(2)
    y, _ = peer.peer_fwd(np.zeros_like(p["x"]), p["q"], p["K1"], p["K2"], p["U"], p["V"], k=2)
    assert np.all(y == 0)
    y, _ = peer.peer_fwd(p["x"], p["q"], p["K1"], p["K2"], np.zeros_like(p["U"]), p["V"], k=2)
    assert np.all(y == 0)


def _loss(p, k):
    y, saved = peer.peer_fwd(p["x"], p["q"], p["K1"], p["K2"], p["U"], p["V"], k)
    return float((y * p["dy"]).sum()), saved


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_finite_differences_all_gradients(seed):
    k = 2
    p = _inputs(seed)
    _, saved = _loss(p, k)
    g = peer.peer_bwd(p["dy"], p["x"], p["q"], p["K1"], p["K2"], p["U"], p["V"], saved)
    N, D = p["V"].shape
    dV = np.zeros((N, D))
    dV[g["rows"]] = g["dV"]
    dU = np.zeros((N, D))
    dU[g["rows"]] = g["dU"]
    analytic = dict(x=g["dx"], q=g["dq"], K1=g["dK1"], K2=g["dK2"], U=dU, V=dV)
    h = 1e-6
    for name, ga in analytic.items():
        fd = np.zeros_like(p[name])
        it = np.nditer(p[name], flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            old = p[name][i]
            p[name][i] = old + h
            lp, sp = _loss(p, k)
            p[name][i] = old - h
            lm, sm = _loss(p, k)
            p[name][i] = old
            assert np.array_equal(sp["idx"], saved["idx"]) and np.array_equal(sm["idx"], saved["idx"])
            fd[i] = (lp - lm) / (2 * h)
        denom = max(np.abs(fd).max(), np.abs(ga).max(), 1e-8)
        assert np.abs(fd - ga).max() / denom < 1e-4, name
