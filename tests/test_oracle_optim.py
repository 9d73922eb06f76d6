"""Pins of oracle/optim.py (SPEC S:506-514 examples)."""
import numpy as np

from oracle import optim
from synthetic import gen


def _state(N, dv, seed):
    V = gen.tensor(seed, "V", (N, dv)).astype(np.float64)
    return V, np.zeros((N, dv)), np.zeros((N, dv)), np.zeros(N, np.int64)


def test_no_rows_touched_leaves_table_unchanged():
    V, m, v, st = _state(16, 4, 0)
    V0 = V.copy()
    optim.sparse_adam_step(V, m, v, st, np.zeros(0, np.int64), np.zeros((0, 4)), lr=0.1)
    assert np.array_equal(V, V0)


def test_every_row_every_step_equals_dense_adam():
    """per-row bias correction == dense Adam when all rows are touched."""
    N, dv = 12, 5
    V, m, v, st = _state(N, dv, 1)
    Vd, md, vd = V.copy(), m.copy(), v.copy()
    for step in range(1, 6):
        g = gen.tensor(step, "dout", (N, dv)).astype(np.float64)
        optim.sparse_adam_step(V, m, v, st, np.arange(N), g, lr=0.05, weight_decay=0.01)
        optim.dense_adam_step(Vd, md, vd, step, g, lr=0.05, weight_decay=0.01)
        np.testing.assert_allclose(V, Vd, rtol=0, atol=1e-14)


def test_first_step_is_sign_step():
    """Closed form: at c = 1, mhat = g and vhat = g^2, so the update is
    lr * g / (|g| + eps) ~ lr * sign(g)."""
    V, m, v, st = _state(4, 3, 2)
    V0 = V.copy()
    g = np.array([[0.5, -2.0, 1e-3]])
    optim.sparse_adam_step(V, m, v, st, np.array([2]), g, lr=0.1, eps=1e-12)
    np.testing.assert_allclose(V[2], V0[2] - 0.1 * np.sign(g[0]), rtol=0, atol=1e-9)
    assert np.array_equal(V[[0, 1, 3]], V0[[0, 1, 3]]) and st.tolist() == [0, 0, 1, 0]


def test_untouched_rows_keep_their_own_step_count():
    V, m, v, st = _state(8, 2, 3)
    g = np.ones((1, 2))
    optim.sparse_adam_step(V, m, v, st, np.array([1]), g, lr=0.01)
    optim.sparse_adam_step(V, m, v, st, np.array([1]), g, lr=0.01)
    optim.sparse_adam_step(V, m, v, st, np.array([5]), g, lr=0.01)
    assert st.tolist() == [0, 2, 0, 0, 0, 1, 0, 0]
