"""Pins of oracle/pkm.py against the paper and SPEC hand examples.

The central pin is the paper's own claim: the two-stage product-key
search returns exactly the top-k of Kq over all N = S^2 concatenated keys.
We check it against a brute force that materialises K (a different
computation: one dot product per full key), on the exact input class (many
exact ties, bit-identical arithmetic) and on continuous inputs.
"""
import json
import os

import numpy as np
import pytest

from oracle import pkm, bag
from synthetic import gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_split_query_example():
    g = GOLD["split_query"]
    q1, q2 = pkm.split_query(np.array(g["q"], float))
    assert q1.tolist() == g["q1"] and q2.tolist() == g["q2"]
    with pytest.raises(ValueError):
        pkm.split_query(np.zeros(5))


@pytest.mark.parametrize("name", ["half_topk_identity", "half_topk_all_equal"])
def test_half_topk_examples(name):
    g = GOLD[name]
    s = pkm.half_scores(np.array(g["q_half"], float), np.array(g["K_half"], float))
    I, sc = pkm.half_topk(s, g["k"])
    assert I.tolist() == g["indices"] and sc.tolist() == g["scores"]


@pytest.mark.parametrize("name", ["combine", "combine_k1"])
def test_combine_examples(name):
    g = GOLD[name]
    flat, sc = pkm.combine_topk(np.array(g["I1"]), np.array(g["s1"], float),
                                np.array(g["I2"]), np.array(g["s2"], float), g["k"], g["S"])
    assert flat.tolist() == g["flat"] and sc.tolist() == g["scores"]


def test_k_greater_than_S_rejected():
    with pytest.raises(ValueError):
        pkm.half_topk(np.zeros(4), 5)


def _tables(seed, S, Dk, cls):
    K1 = gen.tensor(seed, "K1", (S, Dk // 2), cls=cls)
    K2 = gen.tensor(seed, "K2", (S, Dk // 2), cls=cls)
    q = gen.tensor(seed, "q", (Dk,), cls=cls)
    return q.astype(np.float64), K1.astype(np.float64), K2.astype(np.float64)


@pytest.mark.parametrize("S", [4, 16, 64])
@pytest.mark.parametrize("k", [1, 4, 16])
def test_two_stage_equals_materialized_brute_force(S, k):
    """200 seeds per (S, k); exact class bit-identical
    (indices and scores), continuous class identical indices, scores equal
    to rounding."""
    if k > S:
        pytest.skip("k <= sqrt(N)")
    Dk = 8
    for seed in range(200):
        cls = gen.CLS_EXACT if seed % 2 == 0 else gen.CLS_CONTINUOUS
        q, K1, K2 = _tables(seed, S, Dk, cls)
        I_a, s_a = pkm.topk_two_stage(q, K1, K2, k)
        I_b, s_b = pkm.topk_materialized(q, K1, K2, k)
        I_c, s_c = pkm.topk_full(q, K1, K2, k)
        assert I_a.tolist() == I_b.tolist() == I_c.tolist(), (seed, S, k)
        if cls == gen.CLS_EXACT:
            assert s_a.tolist() == s_b.tolist()
        else:
            np.testing.assert_allclose(s_a, s_b, rtol=0, atol=1e-13)


def test_zero_query_selects_first_k():
    """q = 0 -> all scores equal -> indices 0..k-1, w = 1/k."""
    S, Dk, k = 16, 8, 5
    _, K1, K2 = _tables(1, S, Dk, gen.CLS_CONTINUOUS)
    q = np.zeros((1, 1, Dk))
    idx, score, w = pkm.pkm_lookup(q, K1[None], K2[None], k)
    assert idx[0, 0].tolist() == list(range(k))
    np.testing.assert_allclose(w, 1.0 / k, rtol=0, atol=1e-15)


def test_k_equals_N_exhaustive():
    """k = N returns every index, in score order."""
    S, Dk = 4, 6
    q, K1, K2 = _tables(2, S, Dk, gen.CLS_CONTINUOUS)
    I, s = pkm.topk_full(q, K1, K2, S * S)
    assert sorted(I.tolist()) == list(range(S * S))
    assert np.all(np.diff(s) <= 0)


def test_duplicate_keys_distinct_indices():
    """a repeated K1 row still gives distinct flat indices, ties
    broken toward the lower flat index."""
    S, Dk, k = 8, 4, 6
    q, K1, K2 = _tables(3, S, Dk, gen.CLS_CONTINUOUS)
    K1[5] = K1[2]
    I, s = pkm.topk_two_stage(q, K1, K2, k)
    assert len(set(I.tolist())) == k
    Ib, _ = pkm.topk_materialized(q, K1, K2, k)
    assert I.tolist() == Ib.tolist()
    for j in range(k - 1):
        if s[j] == s[j + 1]:
            assert I[j] < I[j + 1]


def test_softmax_examples_and_sum():
    for name in ("softmax_uniform", "softmax_overflow"):
        g = GOLD[name]
        np.testing.assert_allclose(pkm.softmax(np.array(g["x"], float)), g["y"], atol=1e-12)
    x = gen.tensor(4, "q", (50, 7)).astype(np.float64) * 1000
    np.testing.assert_allclose(pkm.softmax(x).sum(-1), 1.0, atol=1e-12)
    # S:59 [1,2,3] vs direct exp/sum (no max subtraction needed there)
    e = np.exp([1.0, 2.0, 3.0])
    np.testing.assert_allclose(pkm.softmax(np.array([1.0, 2.0, 3.0])), e / e.sum(), rtol=1e-15)


def test_lookup_equals_dense_eq1():
    """the composed lookup + bag equals Eq. 1 written literally with a
    materialised K (I = top-k(Kq), s = Softmax(K_I q), y = s V_I)."""
    S, Dk, k, dv = 8, 8, 3, 5
    for seed in range(20):
        q, K1, K2 = _tables(seed, S, Dk, gen.CLS_CONTINUOUS)
        V = gen.tensor(seed, "V", (S * S, dv)).astype(np.float64)
        I, s, y = pkm.dense_eq1(q, K1, K2, V, k)
        idx, score, w = pkm.pkm_lookup(q[None, None], K1[None], K2[None], k)
        yb = bag.embbag_fwd(V, idx.reshape(1, k), w.reshape(1, k))
        assert idx[0, 0].tolist() == I.tolist()
        np.testing.assert_allclose(w[0, 0], s, rtol=1e-13)
        np.testing.assert_allclose(yb[0], y, rtol=1e-13, atol=1e-15)


def test_heads_are_independent():
    """Reading Q1: head h uses only q[:, h] and K1[h], K2[h]."""
    S, Dk, k, H = 8, 6, 3, 3
    q = gen.tensor(5, "q", (4, H, Dk)).astype(np.float64)
    K1 = gen.tensor(5, "K1", (H, S, Dk // 2)).astype(np.float64)
    K2 = gen.tensor(5, "K2", (H, S, Dk // 2)).astype(np.float64)
    idx, score, w = pkm.pkm_lookup(q, K1, K2, k)
    for h in range(H):
        i1, s1, w1 = pkm.pkm_lookup(q[:, h:h + 1], K1[h:h + 1], K2[h:h + 1], k)
        assert np.array_equal(i1[:, 0], idx[:, h])
        np.testing.assert_array_equal(w1[:, 0], w[:, h])


# ------------------------------------------------------------ qk-norm (f2)
def test_qk_norm_scores_bounded_and_parallel_closed_form():
    """with qk_norm every half score lies in [-1, 1]; a query half
    parallel to a key row scores exactly 1 (closed form)."""
    S, Dk, k = 16, 8, 4
    q, K1, K2 = _tables(4, S, Dk, gen.CLS_CONTINUOUS)
    qn, K1n, K2n = pkm._qk(q, K1, K2)
    s1 = K1n @ qn[:Dk // 2]
    assert np.all(np.abs(s1) <= 1 + 1e-12)
    K1p = K1.copy()
    K1p[3] = 2.5 * q[:Dk // 2]
    idx, score, w = pkm.pkm_lookup(q[None, None], K1p[None], K2[None], k, qk_norm=True)
    qn, K1n, K2n = pkm._qk(q, K1p, K2)
    assert abs(K1n[3] @ qn[:Dk // 2] - 1.0) < 1e-12
    assert idx[0, 0, 0] // S == 3          # the parallel key wins half 1


def test_qk_norm_two_stage_equals_brute_force_on_normalised_keys():
    S, Dk, k = 16, 8, 4
    for seed in range(20):
        q, K1, K2 = _tables(seed, S, Dk, gen.CLS_CONTINUOUS)
        idx, score, w = pkm.pkm_lookup(q[None, None], K1[None], K2[None], k, qk_norm=True)
        qn, K1n, K2n = pkm._qk(q, K1, K2)
        Ib, sb = pkm.topk_materialized(qn, K1n, K2n, k)
        assert idx[0, 0].tolist() == Ib.tolist()
        np.testing.assert_allclose(score[0, 0], sb, atol=1e-13)


def test_l2_normalize_bwd_finite_differences():
    x = gen.tensor(5, "q", (3, 6)).astype(np.float64)
    g = gen.tensor(5, "dout", (3, 6)).astype(np.float64)
    an = pkm.l2_normalize_bwd(x, g)
    h = 1e-6
    fd = np.zeros_like(x)
    for i in np.ndindex(x.shape):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        fd[i] = ((pkm.l2_normalize(xp) - pkm.l2_normalize(xm)) * g).sum() / (2 * h)
    np.testing.assert_allclose(an, fd, rtol=1e-6, atol=1e-9)
