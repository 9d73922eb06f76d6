"""GPU parity at the north star's large memories: S = 4096 (C3, 16m keys)
and S = 8192 (C4/C5, 64m keys, the right end of Fig. 1's
memory-size axis).  These shapes leave the S <= 1024 fast paths: the tcgen05
scoring runs S / 256 = 16-32 key subtiles per tile, the half top-k takes the
general bound-and-rank path, and the key/query backward takes the sparse
path.  The oracle is the two-stage search (O3', itself pinned to brute force
on every N <= 2^20 by tests/test_oracle_pkm.py)."""
import numpy as np
import pytest
import torch

from oracle import pkm as opkm
from synthetic import gen
from tests.gpu_util import TOL, assert_close, compare_topk, dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_09764_b200 import ops  # noqa: F401  (fails loudly without the .so)
    yield


def ops():
    from paper_2412_09764_b200 import ops as o
    return o


def _inputs(seed, T, H, S, Dk, cls):
    sc = gen.scale_for("K1", Dk=Dk) if cls == gen.CLS_CONTINUOUS else 1.0
    q = gen.tensor(seed, "q", (T, H, Dk), dtype="bf16", cls=cls)
    K1 = gen.tensor(seed, "K1", (H, S, Dk // 2), scale=sc, dtype="bf16", cls=cls)
    K2 = gen.tensor(seed, "K2", (H, S, Dk // 2), scale=sc, dtype="bf16", cls=cls)
    return q, K1, K2


CASES = [  # (T, H, S, Dk, k): several 128-token tiles + a ragged tail
    (300, 2, 4096, 128, 32),
    (150, 4, 4096, 1024, 32),     # C3 per-head shapes
    (260, 2, 8192, 128, 32),
    (70, 4, 8192, 1024, 32),      # C4 per-head shapes
    (40, 2, 8192, 2048, 16),      # C5 key dim
]


@pytest.mark.parametrize("T,H,S,Dk,k", CASES)
def test_pkm_topk_exact_class_large_S(T, H, S, Dk, k):
    """Exact class: every score exact in fp32 -> indices and scores
    bit-exact, including the many exact ties (lower index wins)."""
    q, K1, K2 = _inputs(31, T, H, S, Dk, gen.CLS_EXACT)
    idx, w, score = ops().pkm_topk(dev(q, "bf16"), dev(K1, "bf16"), dev(K2, "bf16"), k,
                                   with_score=True)
    ridx, rscore, rw = opkm.pkm_lookup(q.astype(np.float64), K1.astype(np.float64),
                                       K2.astype(np.float64), k, method="two_stage")
    assert np.array_equal(host(idx), ridx)
    assert np.array_equal(host(score), rscore)
    assert_close(host(w), rw, 1e-6, "w")


@pytest.mark.parametrize("T,H,S,Dk,k", CASES)
def test_pkm_topk_continuous_large_S(T, H, S, Dk, k):
    q, K1, K2 = _inputs(32, T, H, S, Dk, gen.CLS_CONTINUOUS)
    idx, w, score = ops().pkm_topk(dev(q, "bf16"), dev(K1, "bf16"), dev(K2, "bf16"), k,
                                   with_score=True)
    q64, K164, K264 = (a.astype(np.float64) for a in (q, K1, K2))
    ridx, rscore, rw = opkm.pkm_lookup(q64, K164, K264, k)
    near = compare_topk(host(idx), ridx, q64, K164, K264)
    ok = np.ones(ridx.shape[:2], bool)
    for t, h, _ in near:
        ok[t, h] = False
    assert ok.mean() > 0.98, f"{len(near)} near ties"
    assert_close(host(score)[ok], rscore[ok], 1e-5, "score")
    assert_close(host(w)[ok], rw[ok], TOL["f32"], "w")


@pytest.mark.parametrize("T,H,S,Dk,k", CASES)
def test_pkm_topk_bwd_bf16_large_S(T, H, S, Dk, k):
    """The bf16 key/query backward at large S, element by element vs the
    oracle (the keys are trainable)."""
    q, K1, K2 = _inputs(33, T, H, S, Dk, gen.CLS_CONTINUOUS)
    q64, K164, K264 = (a.astype(np.float64) for a in (q, K1, K2))
    ridx, rscore, rw = opkm.pkm_lookup(q64, K164, K264, k)
    dw = gen.tensor(33, "dout", (T, H, k), dtype="f32")
    rdq, rdK1, rdK2, _ = opkm.pkm_bwd(q64, K164, K264, ridx, rw, dw)
    dq, dK1, dK2 = ops().pkm_topk_bwd(dev(q, "bf16"), dev(K1, "bf16"), dev(K2, "bf16"),
                                      dev(ridx.astype(np.int32)), dev(rw.astype(np.float32)),
                                      dev(dw))
    # products of bf16 inputs accumulated in fp32: the fp32 tolerance holds
    assert_close(host(dq), rdq, TOL["f32"], "dq")
    assert_close(host(dK1), rdK1, TOL["f32"], "dK1")
    assert_close(host(dK2), rdK2, TOL["f32"], "dK2")


def _in_subprocess(q, K1, K2, k, fused, env_extra=None):
    """pkm_topk in a fresh process with the fused scoring + filter kernel
    switched on (ML_PKM_FUSED=1) or off (score matrix + half top-k kernel);
    env_extra: further switches (e.g. ML_TOPK_CHUNKS)."""
    import os, subprocess, sys, tempfile
    with tempfile.TemporaryDirectory() as d:
        np.save(os.path.join(d, "q.npy"), q)
        np.save(os.path.join(d, "K1.npy"), K1)
        np.save(os.path.join(d, "K2.npy"), K2)
        code = (
            "import numpy as np, torch, sys\n"
            "from paper_2412_09764_b200 import ops\n"
            f"d = {d!r}\n"
            "t = lambda n: torch.from_numpy(np.load(d + '/' + n + '.npy')).cuda().to(torch.bfloat16)\n"
            f"i, w, s = ops.pkm_topk(t('q'), t('K1'), t('K2'), {k}, with_score=True)\n"
            "np.save(d + '/i.npy', i.cpu().numpy()); np.save(d + '/w.npy', w.cpu().numpy())\n"
            "np.save(d + '/s.npy', s.cpu().numpy())\n")
        env = dict(os.environ, ML_PKM_FUSED="1" if fused else "0", **(env_extra or {}))
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return (np.load(os.path.join(d, "i.npy")), np.load(os.path.join(d, "w.npy")),
                np.load(os.path.join(d, "s.npy")))


@pytest.mark.parametrize("T,H,S,Dk,k", [(300, 4, 1024, 1024, 32), (260, 2, 8192, 128, 32),
                                        (200, 2, 512, 128, 8), (130, 2, 2048, 256, 1)])
def test_fused_select_equals_score_matrix_path(T, H, S, Dk, k):
    """The fused scoring + threshold filter (no score matrix) selects exactly
    what the score-matrix path selects from the same tensor-core scores:
    indices, scores and weights bit-identical."""
    q, K1, K2 = _inputs(34, T, H, S, Dk, gen.CLS_CONTINUOUS)
    fi, fw, fs = _in_subprocess(q, K1, K2, k, fused=True)
    ui, uw, us = _in_subprocess(q, K1, K2, k, fused=False)
    assert np.array_equal(fi, ui)
    assert np.array_equal(fs, us)
    assert np.array_equal(fw, uw)


def test_fused_select_fallback_rows():
    """Rows whose candidate list overflows (all scores tied: q = 0 on some
    tokens, heavy ties on the exact class) take the exact fallback: q = 0
    selects flat indices 0..k-1 with w = 1/k, the other rows match
    the oracle bit-exactly (exact class)."""
    T, H, S, Dk, k = 96, 2, 1024, 128, 16
    q, K1, K2 = _inputs(35, T, H, S, Dk, gen.CLS_EXACT)
    q[::5] = 0.0
    idx, w, score = _in_subprocess(q, K1, K2, k, fused=True)
    ridx, rscore, rw = opkm.pkm_lookup(q.astype(np.float64), K1.astype(np.float64),
                                       K2.astype(np.float64), k, method="two_stage")
    assert np.array_equal(idx[::5], np.broadcast_to(np.arange(k), (len(q[::5]), H, k)))
    assert np.array_equal(idx, ridx)
    assert np.array_equal(score.astype(np.float64), rscore)
    assert_close(w.astype(np.float64), rw, 1e-6, "w")


@pytest.mark.parametrize("T,H,S,Dk,k,cls", [(300, 2, 4096, 128, 32, gen.CLS_CONTINUOUS),
                                            (260, 2, 8192, 128, 32, gen.CLS_CONTINUOUS),
                                            (130, 2, 2048, 256, 8, gen.CLS_CONTINUOUS),
                                            (200, 2, 4096, 128, 32, gen.CLS_EXACT)])
def test_chunk_filtered_half_topk_equals_streaming(T, H, S, Dk, k, cls):
    """Long rows: the half top-k that reads only the 32-score chunks whose
    maximum (written by the scoring epilogue) reaches the bound selects
    exactly what the two-pass streaming top-k selects: indices, scores and
    weights bit-identical (exact class: heavy ties at the bound)."""
    q, K1, K2 = _inputs(36, T, H, S, Dk, cls)
    ci, cw, cs = _in_subprocess(q, K1, K2, k, fused=False, env_extra={"ML_TOPK_CHUNKS": "1"})
    si, sw, ss = _in_subprocess(q, K1, K2, k, fused=False, env_extra={"ML_TOPK_CHUNKS": "0"})
    assert np.array_equal(ci, si)
    assert np.array_equal(cs, ss)
    assert np.array_equal(cw, sw)
