"""Pins of oracle/bag.py (Eq. 1 "y = s V_I"; §3.1.4).

Second formulation: the bag is the linear map y = A V with the dense
selection matrix A[t, r] = sum_{j: idx[t,j]=r} w[t,j]; then dV = A^T dy
(dense) and dw[t,j] = (dy V^T)[t, idx[t,j]].  Plus the SPEC closed forms.
"""
import json
import os

import numpy as np
import pytest

from oracle import bag
from synthetic import gen, streams

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _V(seed, N, dv):
    return gen.tensor(seed, "V", (N, dv)).astype(np.float64)


def test_selection_identity_and_zero_weights():
    """k=1, w=1 -> the selected row; all-zero weights -> 0."""
    V = _V(0, 32, 6)
    idx = np.array([[3], [31], [0]])
    y = bag.embbag_fwd(V, idx, np.ones((3, 1)))
    assert np.array_equal(y, V[[3, 31, 0]])
    y0 = bag.embbag_fwd(V, streams.uniform_indices(1, 4, 5, 32), np.zeros((4, 5)))
    assert np.all(y0 == 0)


@pytest.mark.parametrize("profile", ["u", "c0", "c50", "c100", "zipf"])
def test_fwd_bwd_equal_dense_formulation(profile):
    N, dv, T, B = 64, 9, 7, 6
    if profile == "u":
        idx = streams.uniform_indices(2, T, B, N)
    elif profile == "zipf":
        idx = streams.zipf_indices(2, T, B, N, 1.1)
    else:
        idx = streams.collision_indices(2, T, B, N, int(profile[1:]))
    w = streams.softmax_free_weights(2, T, B).astype(np.float64)
    V = _V(2, N, dv)
    dy = gen.tensor(2, "dout", (T, dv)).astype(np.float64)
    A = bag.dense_selection_matrix(idx, w, N)
    np.testing.assert_allclose(bag.embbag_fwd(V, idx, w), A @ V, rtol=1e-13, atol=1e-15)
    rows, dV, dw = bag.embbag_bwd(V, idx, w, dy)
    assert rows.tolist() == sorted(set(idx.reshape(-1).tolist()))
    dense = A.T @ dy
    np.testing.assert_allclose(dV, dense[rows], rtol=1e-12, atol=1e-14)
    untouched = np.setdiff1d(np.arange(N), rows)
    assert np.all(dense[untouched] == 0)
    G = dy @ V.T
    np.testing.assert_allclose(dw, np.take_along_axis(G, idx, axis=1), rtol=1e-12, atol=1e-14)


def test_reverse_index_example():
    """indices [[2,2],[5,2]] -> row 2 gets positions (0,0),(0,1),(1,1)
    and row 5 gets (1,0): with w = 1 and one-hot dy rows the dV row of 2 is
    dy[0] + dy[0] + dy[1] and that of 5 is dy[1]."""
    g = GOLD["bag_reverse_index"]
    idx = np.array(g["indices"])
    dy = np.eye(2)
    rows, dV, _ = bag.embbag_bwd(np.zeros((6, 2)), idx, np.ones((2, 2)), dy)
    assert rows.tolist() == [2, 5]
    want2 = sum(dy[t] for t, _ in g["groups"]["2"])
    want5 = sum(dy[t] for t, _ in g["groups"]["5"])
    assert dV[0].tolist() == list(want2) and dV[1].tolist() == list(want5)


def test_linearity():
    N, dv, T, B = 40, 5, 6, 4
    idx = streams.uniform_indices(3, T, B, N)
    w = streams.softmax_free_weights(3, T, B).astype(np.float64)
    V = _V(3, N, dv)
    np.testing.assert_allclose(bag.embbag_fwd(V, idx, 2.5 * w), 2.5 * bag.embbag_fwd(V, idx, w), rtol=1e-14)
    dy = gen.tensor(3, "dout", (T, dv)).astype(np.float64)
    _, dV1, dw1 = bag.embbag_bwd(V, idx, w, dy)
    _, dV3, dw3 = bag.embbag_bwd(V, idx, w, -3 * dy)
    np.testing.assert_allclose(dV3, -3 * dV1, rtol=1e-14)
    np.testing.assert_allclose(dw3, -3 * dw1, rtol=1e-14)


def test_callable_rows_equal_array():
    N, dv = 50, 8
    V = gen.tensor(9, "V", (N, dv), dtype="bf16")
    idx = streams.uniform_indices(9, 5, 3, N)
    w = streams.softmax_free_weights(9, 5, 3)
    a = bag.embbag_fwd(V, idx, w)
    b = bag.embbag_fwd(lambda ids: gen.rows(9, "V", ids, dv, dtype="bf16"), idx, w)
    assert np.array_equal(a, b)


def test_dyadic_class_exact_regardless_of_order():
    """Dyadic weights x bf16-exact values: every partial sum is exact in
    fp64, so any summation order gives the same y (basis of the GPU
    bit-exact bag test)."""
    N, dv, T, B = 64, 16, 8, 12
    V = gen.tensor(4, "V", (N, dv), cls=gen.CLS_EXACT).astype(np.float64)
    idx = streams.uniform_indices(4, T, B, N)
    w = streams.softmax_free_weights(4, T, B, cls=gen.CLS_DYADIC).astype(np.float64)
    y = bag.embbag_fwd(V, idx, w)
    y_rev = bag.embbag_fwd(V, idx[:, ::-1], w[:, ::-1])
    assert np.array_equal(y, y_rev)
