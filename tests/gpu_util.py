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


def assert_close(got, ref, rtol, name="", floor=None):
    """Reading Q17: max|got-ref| <= rtol * max|ref| per tensor (the north_star
    relative tolerance), and elementwise |got-ref| <= rtol * (|ref| +
    floor * max|ref|), floor = 1e-2 for fp32 tolerances and 0.5 for bf16 ones
    (elements that cancel to ~0 carry the rounding of their terms: with bf16
    storage of intermediates that is ~2^-9 of the terms' magnitude)."""
    if floor is None:
        floor = 1e-2 if rtol < 1e-3 else 0.5
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    scale = max(np.abs(ref).max(initial=0.0), 1e-30)
    err = np.abs(got - ref)
    assert err.max(initial=0.0) <= rtol * scale, f"{name}: max err {err.max():.3e} > {rtol} * {scale:.3e}"
    bound = rtol * (np.abs(ref) + floor * scale)
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
