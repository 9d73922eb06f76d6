"""Helpers for the -m gpu parity tests (test infrastructure)."""
import numpy as np
import torch

from oracle import pkm as opkm

TOL = {"f32": 1e-4, "bf16": 2e-2}   # north_star: 1e-4 relative fp32, 2e-2 bf16 (reading Q17)
TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(TORCH_DT[dtype])
    return t.cuda()


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64) if t.dtype != torch.int32 \
        else t.cpu().numpy()


U_BF16 = 2.0 ** -8      # unit roundoff of bf16 storage (8 significant bits, RNE)
KAPPA = 4.0             # bf16 roundings along one element's chain (rounding model)


def assert_close(got, ref, rtol, name="", floor=None, mag=None, u=U_BF16):
    """Reading Q17: max|got-ref| <= rtol * max|ref| per tensor (the north_star
    relative tolerance), and elementwise |got-ref| <= rtol * (|ref| +
    floor * max|ref|), floor = 1e-2 for fp32 tolerances and 0.1 for bf16 ones
    (elements that cancel to ~0 carry the rounding of their terms: with bf16
    storage of intermediates that is ~2^-9 = 2e-3 of the terms' magnitude,
    i.e. ~0.1 * rtol at rtol = 2e-2 when the terms are as large as the
    tensor's largest element)."""
    if floor is None:
        floor = 1e-2 if rtol < 1e-3 else 0.1
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    scale = max(np.abs(ref).max(initial=0.0), 1e-30)
    err = np.abs(got - ref)
    assert err.max(initial=0.0) <= rtol * scale, f"{name}: max err {err.max():.3e} > {rtol} * {scale:.3e}"
    bound = rtol * (np.abs(ref) + floor * scale)
    if mag is not None:
        # rounding model: an element whose terms cancel carries the bf16
        # rounding of its terms, |err| <= KAPPA * u * sum|terms| (mag = that
        # sum, from the oracle on absolute values); u = the unit
        # roundoff of the narrowest intermediate (2^-16 for a bf16 hi/lo pair)
        bound = bound + KAPPA * u * np.asarray(mag, np.float64)
    bad = err > bound
    assert not bad.any(), f"{name}: {bad.sum()} elements beyond elementwise bound; worst {err[bad].max():.3e}"


def flat_score(q, K1h, K2h, flat):
    """fp64 score of flat key a*S+b for one (t,h)."""
    S = K1h.shape[0]
    Dh = K1h.shape[1]
    a, b = np.asarray(flat) // S, np.asarray(flat) % S
    return K1h[a] @ q[:Dh] + K2h[b] @ q[Dh:]


def fp32_bound(q, K1h, K2h, flat):
    """Rigorous fp32 accumulation bound of the kernel's score for flat keys:
    (Dh + 1) * 2^-24 * sum_i |q_i K_i| over both halves (products of bf16 /
    fp32 inputs accumulated in fp32; +1 for the s1 + s2 add)."""
    S = K1h.shape[0]
    Dh = K1h.shape[1]
    a, b = np.asarray(flat) // S, np.asarray(flat) % S
    mag = np.abs(K1h[a]) @ np.abs(q[:Dh]) + np.abs(K2h[b]) @ np.abs(q[Dh:])
    return (Dh + 2) * 2.0 ** -24 * mag


def compare_topk(gpu_idx, ref_idx, q, K1, K2, rel_gap=1e-6):
    """Top-k parity with the near-tie rule (north_star; reading Q18): a
    (t,h) whose GPU index list differs from the oracle's is accepted only if
    every differing slot swaps keys whose fp64 scores are within
    max(rel_gap * |s|, fp32 accumulation bound).  Returns the list of
    accepted near-tie (t,h) and raises on a real mismatch."""
    T, H, k = ref_idx.shape
    near = []
    for t, h in zip(*np.nonzero((gpu_idx != ref_idx).any(-1))):
        g, r = gpu_idx[t, h], ref_idx[t, h]
        assert len(set(g.tolist())) == k, f"duplicate indices at {(t, h)}"
        sg = flat_score(q[t, h], K1[h], K2[h], g)
        sr = flat_score(q[t, h], K1[h], K2[h], r)
        tol = np.maximum(rel_gap * np.maximum(np.abs(sg), np.abs(sr)),
                         fp32_bound(q[t, h], K1[h], K2[h], g) + fp32_bound(q[t, h], K1[h], K2[h], r))
        gap = np.abs(sg - sr)
        assert np.all(gap <= tol), (f"top-k mismatch at (t={t}, h={h}): gpu {g.tolist()} oracle "
                                    f"{r.tolist()} gaps {gap.tolist()} tol {tol.tolist()}")
        near.append((int(t), int(h), float(gap.max())))
    return near


def layer_magnitudes(h, rs, rb, gated=True):
    """Per-element magnitudes sum|terms| of the memory layer's outputs and
    gradients (test infrastructure for the rounding-model bound of
    assert_close): every sum of products of the layer is re-evaluated on the
    absolute values of its factors, with the oracle's selection (rs idx, w)
    and the oracle's intermediates (y, g); silu / its derivative enter as
    absolute values of the real ones.  h: fp64 inputs, rs/rb: the oracle's
    forward saved dict / backward grads."""
    from oracle import gate as ogate
    A = np.abs
    T, H, k = rs["idx"].shape
    S = h["K1"].shape[1]
    Dh = h["K1"].shape[2]
    B = H * k
    idx = rs["idx"].reshape(T, B)
    w = A(rs["w"]).reshape(T, B)
    V = h["V"]
    m = {}
    if gated:
        g, y = rs["g"], rs["y"]
        sg = A(ogate.silu(g))
        z = A(y) * sg
        m["out"] = z @ A(h["W2"])
        mdz = A(h["dout"]) @ A(h["W2"]).T
        mdy = mdz * sg
        mdg = mdz * A(y) * A(ogate.dsilu(g))
        m["dx"] = mdg @ A(h["W1"]).T
        m["dW1"] = A(h["x"]).T @ mdg
        m["dW2"] = z.T @ A(h["dout"])
    else:
        mdy = A(h["dout"])
        m["out"] = np.einsum("tj,tjc->tc", w, A(V[idx]))
    m["y"] = np.einsum("tj,tjc->tc", w, A(V[idx]))
    mdw = np.einsum("tc,tjc->tj", mdy, A(V[idx]))
    m["dw"] = mdw.reshape(T, H, k)
    rows = rb["rows"]
    pos = {int(r): i for i, r in enumerate(rows)}
    mdV = np.zeros((len(rows), V.shape[1]))
    for t in range(T):
        for j in range(B):
            mdV[pos[int(idx[t, j])]] += w[t, j] * mdy[t]
    m["dV"] = mdV
    m["dq"], m["dK1"], m["dK2"] = key_magnitudes(h["q"], h["K1"], h["K2"], rs["idx"], rs["w"],
                                                 mdw.reshape(T, H, k))
    return m


def key_magnitudes(q, K1, K2, idx, w, mdw):
    """sum|terms| of dq, dK1, dK2 (PAPER.md P:145 key backward) given the
    selection (idx, w) and the magnitudes of dw: ds magnitudes
    |w| (|dw| + sum_j |w_j||dw_j|), then the two contractions on absolute
    values."""
    A = np.abs
    T, H, k = idx.shape
    S, Dh = K1.shape[1], K1.shape[2]
    mw = A(mdw)
    wk = A(w)
    mds = wk * (mw + (wk * mw).sum(-1, keepdims=True))
    h = {"q": q, "K1": K1, "K2": K2}
    rs = {"idx": idx}
    mdq = np.zeros((T, H, 2 * Dh))
    mdK1 = np.zeros(h["K1"].shape)
    mdK2 = np.zeros(h["K2"].shape)
    a, b = rs["idx"] // S, rs["idx"] % S
    q = A(h["q"])
    for hh in range(H):
        for j in range(k):
            mdq[:, hh, :Dh] += mds[:, hh, j, None] * A(h["K1"][hh, a[:, hh, j]])
            mdq[:, hh, Dh:] += mds[:, hh, j, None] * A(h["K2"][hh, b[:, hh, j]])
            np.add.at(mdK1[hh], a[:, hh, j], mds[:, hh, j, None] * q[:, hh, :Dh])
            np.add.at(mdK2[hh], b[:, hh, j], mds[:, hh, j, None] * q[:, hh, Dh:])
    return mdq, mdK1, mdK2
