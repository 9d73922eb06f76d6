"""PEER-style rank-1 expert retrieval over product keys:
the adjacent method the paper compares against ("replacing
vector values with rank-one matrices", "it retrieves a pair of
embeddings, which combine into a rank-1 matrix.  Several of these are
assembled together into a dynamic feed-forward layer").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reading Q21 (the paper gives no formula): key i owns a pair
(U[i], V[i]), U, V in R^{N x D}.  The same product-key lookup as the memory
layer (pkm.pkm_lookup: idx, softmax weights w over the k selected keys of
each head) selects the experts; expert i applied to token x is the rank-1
map x -> silu(U[i] . x) V[i] (activation: silu, as in the Memory+ gate,
P:191); the layer output sums the heads' experts weighted by w:

    h[t, j] = U[idx[t, j]] . x[t]
    a[t, j] = w[t, j] * silu(h[t, j])
    y[t]    = sum_j a[t, j] V[idx[t, j]]

float64 throughout.
"""
import numpy as np

from . import pkm, bag, gate


def peer_fwd(x, q, K1, K2, U, V, k, qk_norm=False):
    """Returns y [T, D] and the saved tensors (idx, w, h, a)."""
    T, H, _ = q.shape
    idx, score, w = pkm.pkm_lookup(q, K1, K2, k, qk_norm=qk_norm)
    bidx = idx.reshape(T, H * k)
    bw = w.reshape(T, H * k)
    x = np.asarray(x, np.float64)
    Ur = np.asarray(U, np.float64)
    h = np.einsum("tjd,td->tj", Ur[bidx], x)
    a = bw * gate.silu(h)
    y = bag.embbag_fwd(V, bidx, a)
    return y, dict(idx=idx, w=w, h=h, a=a, qk_norm=qk_norm)


def peer_bwd(dy, x, q, K1, K2, U, V, saved):
    """Chain rule of peer_fwd given dy [T, D]:
        (rows, dV, da) = embbag_bwd(V, idx, a, dy)       da[t,j] = <dy[t], V[idx]>
        dh  = da * w * silu'(h)
        dwr = da * silu(h)                                 (router weights)
        dU[r] = sum_{p: idx[p] = r} dh[p] x[t(p)]          (same rows as dV)
        dx[t] = sum_j dh[t, j] U[idx[t, j]]
        dq, dK1, dK2 = pkm_bwd(..., dw = dwr)
    Returns a dict with rows, dV, dU (both [U_rows, D], rows ascending), dx,
    dq, dK1, dK2, dwr, dh."""
    idx, w, h = saved["idx"], saved["w"], saved["h"]
    T, H, k = idx.shape
    bidx = idx.reshape(T, H * k)
    bw = w.reshape(T, H * k)
    x = np.asarray(x, np.float64)
    rows, dV, da = bag.embbag_bwd(V, bidx, saved["a"], dy)
    dh = da * bw * gate.dsilu(h)
    dwr = da * gate.silu(h)
    rows_u, dU, _ = bag.embbag_bwd(U, bidx, dh, x)
    assert np.array_equal(rows_u, rows)
    dx = bag.embbag_fwd(U, bidx, dh)
    dq, dK1, dK2, ds = pkm.pkm_bwd(q, K1, K2, idx, w, dwr.reshape(T, H, k),
                                   qk_norm=saved.get("qk_norm", False))
    return dict(rows=rows, dV=dV, dU=dU, dx=dx, dq=dq, dK1=dK1, dK2=dK2,
                dwr=dwr.reshape(T, H, k), dh=dh.reshape(T, H, k))
