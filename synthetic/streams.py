"""Index / weight streams for the bag-only parity tests.

U: uniform rows; Z(alpha): Zipf ranks mapped to rows by an odd-multiplier
bijection mod N; C(c): collision profiles (c % of positions drawn from a
small hot set, the rest distinct) as in SPEC.md S:284.  None of this is
method arithmetic: these are inputs.
"""
import numpy as np

from .gen import counter_u64, unit_values, TAGS, CLS_CONTINUOUS, CLS_DYADIC


def uniform_indices(seed, T, B, N):
    u = counter_u64(seed, TAGS["idx"], np.arange(T * B, dtype=np.uint64))
    return (u % np.uint64(N)).astype(np.int32).reshape(T, B)


def zipf_indices(seed, T, B, N, alpha):
    """Zipf(alpha) over ranks 1..N via inverse CDF on a fp64 table; rank r
    maps to row (r * 0x9E3779B1) mod N (odd multiplier => bijection when N is
    a power of two; for other N we fall back to r mod N)."""
    u = counter_u64(seed, TAGS["idx"], np.arange(T * B, dtype=np.uint64))
    p = (u >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    ranks = np.arange(1, N + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** (-alpha))
    cdf /= cdf[-1]
    r = np.searchsorted(cdf, p, side="right").astype(np.uint64)
    r = np.minimum(r, np.uint64(N - 1))
    if N & (N - 1) == 0:
        rows = (r * np.uint64(0x9E3779B1)) & np.uint64(N - 1)
    else:
        rows = r % np.uint64(N)
    return rows.astype(np.int32).reshape(T, B)


def collision_indices(seed, T, B, N, percent):
    """`percent`% of the T*B positions hit one hot row (row 0 of a permuted
    order); the rest get distinct rows (requires T*B <= N for 0%)."""
    P = T * B
    u = counter_u64(seed, TAGS["idx"], np.arange(P, dtype=np.uint64))
    perm_key = u.argsort(kind="stable")
    distinct = (np.arange(P, dtype=np.int64) * 2654435761) % N
    out = distinct.copy()
    n_hot = (P * percent) // 100
    hot_pos = perm_key[:n_hot]
    out[hot_pos] = int(u[0] % np.uint64(N))
    return out.astype(np.int32).reshape(T, B)


def softmax_free_weights(seed, T, B, cls=CLS_CONTINUOUS):
    """Positive bag weights (not a softmax): continuous |f| in [0,1) or
    dyadic multiples of 1/64."""
    u = counter_u64(seed, TAGS["w"], np.arange(T * B, dtype=np.uint64))
    f = unit_values(u, cls)
    if cls == CLS_CONTINUOUS:
        f = np.abs(f)
    return f.astype(np.float32).reshape(T, B)


__all__ = ["uniform_indices", "zipf_indices", "collision_indices",
           "softmax_free_weights", "CLS_DYADIC"]
