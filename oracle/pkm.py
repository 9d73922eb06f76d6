"""Product-key lookup (§3.1.1; Eq. 1).

Reading of the paper used here:
* Q1 heads: H independent heads, each with its own query slice q[t,h,:] and
  its own half-key tables K1[h], K2[h]; a softmax per head.
* Q5 flat index i = a*S + b (S = sqrt(N)); order = score descending, ties to
  the lower index (half top-k: lower sub-index; combined: lower flat index).
* Q4 no temperature: w = softmax(s) over the k selected scores.
* Q8 no gradient through the selection itself.

All arithmetic is float64.
"""
import numpy as np


QK_EPS = 1e-6


def l2_normalize(x, eps=QK_EPS):
    """qk-normalization ("We use qk-normalization when needed"; form
    unspecified -- reading Q12 / SPEC S:193: L2 normalisation of each query
    half and each half-key row at score time, non-learned):
    x / max(||x||_2, eps) over the last axis."""
    x = np.asarray(x, np.float64)
    n = np.sqrt((x * x).sum(axis=-1, keepdims=True))
    return x / np.maximum(n, eps)


def l2_normalize_bwd(x, g, eps=QK_EPS):
    """Gradient of l2_normalize at x given dL/dy = g:
    (g - y (y.g)) / ||x|| when ||x|| > eps, else g / eps."""
    x = np.asarray(x, np.float64)
    g = np.asarray(g, np.float64)
    n = np.sqrt((x * x).sum(axis=-1, keepdims=True))
    y = x / np.maximum(n, eps)
    proj = (g - y * (y * g).sum(axis=-1, keepdims=True)) / np.maximum(n, eps)
    return np.where(n > eps, proj, g / eps)


def _qk(q, K1, K2):
    """Per-half normalised query [.., Dk] and half-key tables."""
    q1, q2 = split_query(q)
    return np.concatenate([l2_normalize(q1), l2_normalize(q2)], axis=-1), l2_normalize(K1), l2_normalize(K2)


def split_query(q):
    """P:157 "we first split the query as q1, q2 in R^{n/2}": first half,
    second half."""
    n = q.shape[-1]
    if n % 2:
        raise ValueError("odd query dimension (S:143)")
    return q[..., : n // 2], q[..., n // 2:]


def order_desc(scores, ids):
    """Permutation sorting by (score descending, id ascending) (Q5)."""
    return np.lexsort((np.asarray(ids), -np.asarray(scores, dtype=np.float64)))


def half_scores(q_half, K_half):
    """scores of one query half against the sqrt(N) half keys,
    s[a] = sum_i q_half[i] * K_half[a, i]."""
    return np.asarray(K_half, np.float64) @ np.asarray(q_half, np.float64)


def half_topk(s, k):
    """P:157 "Let I1, I2 and s1, s2 be the top-k indices and scores obtained
    from the respective key sets"; requires k <= sqrt(N)."""
    S = s.shape[0]
    if not 1 <= k <= S:
        raise ValueError("need 1 <= k <= sqrt(N) (S:150)")
    o = order_desc(s, np.arange(S))[:k]
    return o, s[o]


def combine_topk(I1, s1, I2, s2, k, S):
    """P:157 "The overall indices and scores can be found by taking
    argmax_{i1 in I1, i2 in I2} s1[i1] + s2[i2]": the k best of the k*k
    Cartesian sums, flat index I1*S + I2."""
    cand = (s1[:, None] + s2[None, :]).reshape(-1)
    flat = (np.asarray(I1, np.int64)[:, None] * S
            + np.asarray(I2, np.int64)[None, :]).reshape(-1)
    o = order_desc(cand, flat)[:k]
    return flat[o], cand[o]


def topk_two_stage(q, K1h, K2h, k):
    """The paper's product-key algorithm for one (token, head) (O3')."""
    S = K1h.shape[0]
    q1, q2 = split_query(q)
    I1, s1 = half_topk(half_scores(q1, K1h), k)
    I2, s2 = half_topk(half_scores(q2, K2h), k)
    return combine_topk(I1, s1, I2, s2, k, S)


def topk_full(q, K1h, K2h, k):
    """Eq. 1 "I = SelectTopkIndices(Kq)" over all N = S^2 virtual keys (O3).
    Row a*S+b of the never-instantiated K is concat(K1[a], K2[b]), so
    its score is q1.K1[a] + q2.K2[b]; all N scores, one full sort."""
    S = K1h.shape[0]
    q1, q2 = split_query(q)
    s1, s2 = half_scores(q1, K1h), half_scores(q2, K2h)
    scores = (s1[:, None] + s2[None, :]).reshape(-1)
    flat = np.arange(S * S, dtype=np.int64)
    o = order_desc(scores, flat)[:k]
    return flat[o], scores[o]


def topk_materialized(q, K1h, K2h, k):
    """Brute force that DOES instantiate the full key matrix K in R^{N x n}
    ("The full set of keys ... consists of the product of these two
    sets"), computes Kq and sorts.  Tiny tables only."""
    S = K1h.shape[0]
    if S * S * (K1h.shape[1] * 2) > 1 << 24:
        raise ValueError("materialised brute force is for tiny tables only")
    K = np.concatenate([np.repeat(K1h, S, axis=0), np.tile(K2h, (S, 1))], axis=1)
    scores = np.asarray(K, np.float64) @ np.asarray(q, np.float64)
    flat = np.arange(S * S, dtype=np.int64)
    o = order_desc(scores, flat)[:k]
    return flat[o], scores[o]


def softmax(s):
    """Eq. 1 "s = Softmax(K_I q)", with max subtraction, last axis."""
    s = np.asarray(s, np.float64)
    m = s.max(axis=-1, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(axis=-1, keepdims=True)


def pkm_lookup(q, K1, K2, k, method="two_stage", qk_norm=False):
    """Eq. 1 lookup for every token and head.

    q: [T, H, Dk]; K1, K2: [H, S, Dk/2].  Returns idx [T,H,k] (int64 flat
    index a*S+b), score [T,H,k] (pre-softmax, = K_I q) and w [T,H,k]
    (softmax per head).  qk_norm: the query halves and half-key rows are
    L2-normalised first (l2_normalize)."""
    if qk_norm:
        q, K1, K2 = _qk(q, K1, K2)
    T, H, _ = q.shape
    f = {"two_stage": topk_two_stage, "full": topk_full,
         "materialized": topk_materialized}[method]
    idx = np.zeros((T, H, k), np.int64)
    score = np.zeros((T, H, k), np.float64)
    for t in range(T):
        for h in range(H):
            idx[t, h], score[t, h] = f(q[t, h], K1[h], K2[h], k)
    return idx, score, softmax(score)


def dense_eq1(q, K1h, K2h, V, k):
    """Eq. 1 written literally for one query: materialise K, I = top-k of Kq,
    s = Softmax(K_I q), y = s V_I.  Tiny tables only."""
    S = K1h.shape[0]
    K = np.concatenate([np.repeat(K1h, S, axis=0), np.tile(K2h, (S, 1))], axis=1)
    Kq = np.asarray(K, np.float64) @ np.asarray(q, np.float64)
    I = order_desc(Kq, np.arange(S * S))[:k]
    s = softmax(K[I] @ q)
    return I, s, s @ np.asarray(V, np.float64)[I]


def pkm_bwd(q, K1, K2, idx, w, dw, qk_norm=False):
    """Backward of the lookup into the query and the half keys ("the
    keys and values ... are trainable parameters").

    Softmax backward: ds_j = w_j (dw_j - sum_l w_l dw_l).  The selected
    score is s_j = q1.K1[h, a_j] + q2.K2[h, b_j] with a_j = idx // S,
    b_j = idx % S, hence dq1 = sum_j ds_j K1[h, a_j], dK1[h, a_j] += ds_j q1
    (and the same for half 2).  No gradient through the selection (Q8).
    Returns dq [T,H,Dk], dK1, dK2 [H,S,Dk/2].  With qk_norm the same is done
    for the normalised operands and chained through l2_normalize_bwd."""
    if qk_norm:
        qn, K1n, K2n = _qk(q, K1, K2)
        dqn, dK1n, dK2n, ds = pkm_bwd(qn, K1n, K2n, idx, w, dw)
        Dh = q.shape[-1] // 2
        dq = np.concatenate([l2_normalize_bwd(q[..., :Dh], dqn[..., :Dh]),
                             l2_normalize_bwd(q[..., Dh:], dqn[..., Dh:])], axis=-1)
        return dq, l2_normalize_bwd(K1, dK1n), l2_normalize_bwd(K2, dK2n), ds
    T, H, Dk = q.shape
    S = K1.shape[1]
    Dh = Dk // 2
    w = np.asarray(w, np.float64)
    dw = np.asarray(dw, np.float64)
    ds = w * (dw - (w * dw).sum(axis=-1, keepdims=True))
    a = idx // S
    b = idx % S
    dq = np.zeros((T, H, Dk))
    dK1 = np.zeros(K1.shape)
    dK2 = np.zeros(K2.shape)
    for t in range(T):
        for h in range(H):
            dq[t, h, :Dh] = ds[t, h] @ K1[h, a[t, h]]
            dq[t, h, Dh:] = ds[t, h] @ K2[h, b[t, h]]
            np.add.at(dK1[h], a[t, h], ds[t, h][:, None] * q[t, h, :Dh][None, :])
            np.add.at(dK2[h], b[t, h], ds[t, h][:, None] * q[t, h, Dh:][None, :])
    return dq, dK1, dK2, ds
