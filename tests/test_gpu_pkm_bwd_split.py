"""The opt-in split form of the tcgen05 key/query backward
(ML_PKM_BWD_SPLIT=1): the selected score gradients ds go to
the tensor cores as a bf16 pair hi + lo (hi = RN(ds), lo = RN(ds - hi)), so
dq and dK carry ~16 significant bits of ds instead of 8.  Against the oracle
(the keys are trainable) the fp32 tolerance holds, where the
single-bf16 form needs the bf16 bound.  Runs in a fresh process because the
switch is read once per process."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch

from oracle import pkm as opkm
from synthetic import gen
from tests.gpu_util import TOL, assert_close, key_magnitudes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_09764_b200 import ops  # noqa: F401  (fails loudly without the .so)
    yield


# the key-backward form under test is set explicitly, whatever the outer
# environment selects (the suite is also run under these switches)
_FORM = {"ML_PKM_BWD_SPARSE": "0", "ML_PKM_BWD_SPLIT": "0", "ML_PKM_BWD_F16": "0",
         "ML_PKM_BWD_TC": "1"}


def _bwd_in_subprocess(arrays, split):
    with tempfile.TemporaryDirectory() as d:
        for n, a in arrays.items():
            np.save(os.path.join(d, n + ".npy"), a)
        code = (
            "import numpy as np, torch\n"
            "from paper_2412_09764_b200 import ops\n"
            f"d = {d!r}\n"
            "L = lambda n: torch.from_numpy(np.load(d + '/' + n + '.npy')).cuda()\n"
            "b = lambda n: L(n).to(torch.bfloat16)\n"
            "dq, dK1, dK2 = ops.pkm_topk_bwd(b('q'), b('K1'), b('K2'), L('idx'), L('w'), L('dw'))\n"
            "for n, t in (('dq', dq), ('dK1', dK1), ('dK2', dK2)):\n"
            "    np.save(d + '/o_' + n + '.npy', t.float().cpu().numpy())\n")
        env = {**os.environ, **_FORM, "ML_PKM_BWD_SPLIT": "1" if split else "0"}
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return [np.load(os.path.join(d, f"o_{n}.npy")) for n in ("dq", "dK1", "dK2")]


CASES = [  # (T, H, S, Dk, k): several 128-row tiles + a ragged tail, BN = 64 / 128 / 256
    (300, 4, 1024, 1024, 32),     # C2 per-head shapes
    (150, 2, 512, 128, 8),
    (200, 2, 2048, 256, 16),
]


@pytest.mark.parametrize("T,H,S,Dk,k", CASES)
def test_split_ds_backward_meets_fp32_tolerance(T, H, S, Dk, k):
    sc = gen.scale_for("K1", Dk=Dk)
    q = gen.tensor(41, "q", (T, H, Dk), dtype="bf16")
    K1 = gen.tensor(41, "K1", (H, S, Dk // 2), scale=sc, dtype="bf16")
    K2 = gen.tensor(41, "K2", (H, S, Dk // 2), scale=sc, dtype="bf16")
    q64, K164, K264 = (a.astype(np.float64) for a in (q, K1, K2))
    ridx, _, rw = opkm.pkm_lookup(q64, K164, K264, k)
    dw = gen.tensor(41, "dout", (T, H, k), dtype="f32")
    rdq, rdK1, rdK2, _ = opkm.pkm_bwd(q64, K164, K264, ridx, rw, dw)
    arrays = dict(q=q.astype(np.float32), K1=K1.astype(np.float32), K2=K2.astype(np.float32),
                  idx=ridx.astype(np.int32), w=rw.astype(np.float32), dw=dw.astype(np.float32))
    dq, dK1, dK2 = _bwd_in_subprocess(arrays, split=True)
    # elementwise: the rounding model with u = 2^-16 (the pair's precision,
    # DESIGN.md §3 / §7) on sum|terms| of each element
    mdq, mdK1, mdK2 = key_magnitudes(q64, K164, K264, ridx, rw, dw)
    assert_close(dq, rdq, TOL["f32"], "dq", mag=mdq, u=2.0 ** -16)
    assert_close(dK1, rdK1, TOL["f32"], "dK1", mag=mdK1, u=2.0 ** -16)
    assert_close(dK2, rdK2, TOL["f32"], "dK2", mag=mdK2, u=2.0 ** -16)
    # the single-bf16 form: the bf16 rounding model; the split is closer
    sq, sK1, _ = _bwd_in_subprocess(arrays, split=False)
    assert_close(sq, rdq, TOL["bf16"], "dq (bf16 ds)", mag=mdq)
    assert_close(sK1, rdK1, TOL["bf16"], "dK1 (bf16 ds)", mag=mdK1)
    rel = lambda a, r: float(np.max(np.abs(a - r)) / np.max(np.abs(r)))
    print(f"max rel err dq: split {rel(dq, rdq):.2e}, bf16 ds {rel(sq, rdq):.2e}; "
          f"dK1: split {rel(dK1, rdK1):.2e}, bf16 ds {rel(sK1, rdK1):.2e}")
    assert rel(dq, rdq) < rel(sq, rdq) and rel(dK1, rdK1) < rel(sK1, rdK1)


def _bwd_env(arrays, env):
    with tempfile.TemporaryDirectory() as d:
        for n, a in arrays.items():
            np.save(os.path.join(d, n + ".npy"), a)
        code = (
            "import numpy as np, torch\n"
            "from paper_2412_09764_b200 import ops\n"
            f"d = {d!r}\n"
            "L = lambda n: torch.from_numpy(np.load(d + '/' + n + '.npy')).cuda()\n"
            "b = lambda n: L(n).to(torch.bfloat16)\n"
            "dq, dK1, dK2 = ops.pkm_topk_bwd(b('q'), b('K1'), b('K2'), L('idx'), L('w'), L('dw'))\n"
            "for n, t in (('dq', dq), ('dK1', dK1), ('dK2', dK2)):\n"
            "    np.save(d + '/o_' + n + '.npy', t.float().cpu().numpy())\n")
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **_FORM, **env},
                           cwd=root, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return [np.load(os.path.join(d, f"o_{n}.npy")) for n in ("dq", "dK1", "dK2")]


@pytest.mark.parametrize("T,H,S,Dk,k", [(300, 2, 512, 512, 16), (130, 4, 1024, 1024, 32)])
def test_cta_pair_backward_equals_single_cta(T, H, S, Dk, k):
    """The CTA-pair (cta_group::2, M = 256) key/query backward GEMMs give
    exactly the single-CTA kernels' dq / dK (same k-step order per element),
    including a ragged token count whose last pair has an empty half."""
    sc = gen.scale_for("K1", Dk=Dk)
    q = gen.tensor(42, "q", (T, H, Dk), dtype="bf16")
    K1 = gen.tensor(42, "K1", (H, S, Dk // 2), scale=sc, dtype="bf16")
    K2 = gen.tensor(42, "K2", (H, S, Dk // 2), scale=sc, dtype="bf16")
    ridx, _, rw = opkm.pkm_lookup(q.astype(np.float64), K1.astype(np.float64), K2.astype(np.float64), k)
    dw = gen.tensor(42, "dout", (T, H, k), dtype="f32")
    arrays = dict(q=q.astype(np.float32), K1=K1.astype(np.float32), K2=K2.astype(np.float32),
                  idx=ridx.astype(np.int32), w=rw.astype(np.float32), dw=dw.astype(np.float32))
    pair = _bwd_env(arrays, {"ML_PKM_BWD_PAIR": "1"})
    single = _bwd_env(arrays, {"ML_PKM_BWD_PAIR": "0"})
    for a, b in zip(pair, single):
        assert np.array_equal(a, b)


def _case(seed, T, H, S, Dk, k, dw_scale=1.0, q_scale=1.0, k_scale=1.0):
    # q_scale / k_scale: powers of two (the bf16 values stay exact)
    sc = gen.scale_for("K1", Dk=Dk)
    q = gen.tensor(seed, "q", (T, H, Dk), dtype="bf16") * q_scale
    K1 = gen.tensor(seed, "K1", (H, S, Dk // 2), scale=sc, dtype="bf16") * k_scale
    K2 = gen.tensor(seed, "K2", (H, S, Dk // 2), scale=sc, dtype="bf16") * k_scale
    q64, K164, K264 = (a.astype(np.float64) for a in (q, K1, K2))
    ridx, _, rw = opkm.pkm_lookup(q64, K164, K264, k)
    dw = gen.tensor(seed, "dout", (T, H, k), dtype="f32").astype(np.float64) * dw_scale
    dw = dw.astype(np.float32)
    ref = opkm.pkm_bwd(q64, K164, K264, ridx, rw, dw.astype(np.float64))[:3]
    arrays = dict(q=q.astype(np.float32), K1=K1.astype(np.float32), K2=K2.astype(np.float32),
                  idx=ridx.astype(np.int32), w=rw.astype(np.float32), dw=dw)
    return arrays, ref, key_magnitudes(q64, K164, K264, ridx, rw, dw.astype(np.float64))


@pytest.mark.parametrize("T,H,S,Dk,k,dw_scale,q_scale,k_scale", [
    (300, 4, 1024, 1024, 32, 1.0, 1.0, 1.0),    # C2 per-head shapes (CTA-pair kernels)
    (150, 2, 512, 128, 8, 1.0, 1.0, 1.0),       # single-CTA kernels (BN = 64)
    (130, 4, 1024, 1024, 32, 1e-30, 1.0, 1.0),  # the 2^e scale keeps tiny gradients normal in fp16
    (130, 2, 1024, 512, 16, 1e25, 1.0, 1.0),    # ... and huge ones finite
    (130, 2, 1024, 512, 16, 1.0, 2.0 ** 20, 2.0 ** -12),   # q beyond fp16's range, tiny keys:
    (130, 2, 512, 256, 16, 1.0, 2.0 ** -24, 2.0 ** 18),    # the rescaling second pass
])
def test_fp16_ds_backward_meets_1e3(T, H, S, Dk, k, dw_scale, q_scale, k_scale):
    """The opt-in fp16 form (ML_PKM_BWD_F16=1) of the tcgen05 key/query
    backward runs on fp16 operands, each
    scaled by a power of two from a bound on its magnitude: ds (11
    significant bits instead of bf16's 8) and exact copies of the bf16 q /
    keys; the epilogue unscales: dq, dK1, dK2 within 1e-3 of the fp64 oracle
    (max error / max |ref|), elementwise within the rounding model at
    u = 2^-11; the bf16 ds (ML_PKM_BWD_F16=0) is strictly worse."""
    arrays, (rdq, rdK1, rdK2), (mdq, mdK1, mdK2) = _case(43, T, H, S, Dk, k, dw_scale, q_scale, k_scale)
    got = _bwd_env(arrays, {"ML_PKM_BWD_F16": "1"})
    rel = lambda a, r: float(np.max(np.abs(a - r)) / np.max(np.abs(r)))
    for g, r, m, n in zip(got, (rdq, rdK1, rdK2), (mdq, mdK1, mdK2), ("dq", "dK1", "dK2")):
        assert np.all(np.isfinite(g)), n
        assert rel(g, r) <= 1e-3, (n, rel(g, r))
        assert_close(g, r, 1e-3, n, mag=m, u=2.0 ** -11)
    if dw_scale == 1.0 and q_scale == 1.0:
        old = _bwd_env(arrays, {"ML_PKM_BWD_F16": "0"})
        print("max rel err fp16 ds / bf16 ds:",
              [f"{rel(g, r):.2e} / {rel(o, r):.2e}" for g, o, r in zip(got, old, (rdq, rdK1, rdK2))])
        assert all(rel(g, r) < rel(o, r) for g, o, r in zip(got, old, (rdq, rdK1, rdK2)))
