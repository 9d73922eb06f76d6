"""EmbeddingBag forward and backward (Eq. 1 "y = s V_I"; PAPER.md
§3.1.4).

One bag per token holds B = H*k (index, weight) pairs: the heads' selections
are summed into one output row (reading Q1).  `V` may be an array [N, dv] or
a callable `V(ids) -> [len(ids), dv]` that regenerates rows on demand, so
full-size tables never need to exist on the host.  float64 throughout.
"""
import numpy as np


def _rows(V, ids):
    ids = np.asarray(ids, np.int64)
    if callable(V):
        return np.asarray(V(ids), np.float64)
    return np.asarray(V, np.float64)[ids]


def embbag_fwd(V, idx, w):
    """y[t, :] = sum_j w[t, j] * V[idx[t, j], :]  (Eq. 1).
    idx, w: [T, B]."""
    T, B = idx.shape
    out = None
    for t in range(T):
        r = _rows(V, idx[t])
        yt = np.asarray(w[t], np.float64) @ r
        if out is None:
            out = np.zeros((T, r.shape[1]))
        out[t] = yt
    if out is None:
        raise ValueError("empty batch")
    return out


def embbag_bwd(V, idx, w, dy):
    """Gradients of y = sum_j w_j V[idx_j]:

    dV[r, :] = sum over positions p with idx[p] == r of w[p] * dy[t(p), :]
    (sequential scatter-add in position order; the touched rows are exactly
    the distinct indices, returned ascending as a SparseGrad);
    dw[t, j]  = <dy[t, :], V[idx[t, j], :]>.
    Returns rows [U], dV [U, dv], dw [T, B]."""
    T, B = idx.shape
    dy = np.asarray(dy, np.float64)
    rows, inv = np.unique(np.asarray(idx, np.int64).reshape(-1), return_inverse=True)
    inv = inv.reshape(T, B)
    dV = np.zeros((rows.shape[0], dy.shape[1]))
    dw = np.zeros((T, B))
    for t in range(T):
        np.add.at(dV, inv[t], np.asarray(w[t], np.float64)[:, None] * dy[t][None, :])
        dw[t] = _rows(V, idx[t]) @ dy[t]
    return rows, dV, dw


def dense_selection_matrix(idx, w, N):
    """A [T, N] with A[t, r] = sum_{j: idx[t,j] = r} w[t, j]: the bag as a
    dense linear map, y = A V and dV_dense = A^T dy.  Tiny N only; a second
    formulation used to pin embbag_fwd / embbag_bwd."""
    T, B = idx.shape
    A = np.zeros((T, N))
    for t in range(T):
        for j in range(B):
            A[t, idx[t, j]] += w[t, j]
    return A
