"""shared memory pool across layers -- the value
gradient of 3 layers in one sorted pass -- and the fused-input sparse Adam
 consuming the compact gradient, vs the oracle."""
import numpy as np
import pytest
import torch

from oracle import bag as obag, optim as ooptim
from synthetic import gen, streams
from tests.gpu_util import TOL, assert_close, dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _layers(L, T, B, N, dv, dtype):
    out = []
    for l in range(L):
        idx = streams.zipf_indices(20 + l, T, B, N, 0.9)
        w = streams.softmax_free_weights(20 + l, T, B)
        dy = gen.tensor(20 + l, "dout", (T, dv), dtype=dtype)
        out.append((idx, w, dy))
    return out


@pytest.mark.parametrize("dtype,dv", [("f32", 64), ("bf16", 512)])
def test_shared_pool_three_layers(dtype, dv):
    from paper_2412_09764_b200 import ops
    L, T, B, N = 3, 50, 24, 2048
    V = gen.tensor(9, "V", (N, dv), dtype=dtype)
    lay = _layers(L, T, B, N, dv, dtype)
    rows, dV, U, dws = ops.embbag_bwd_pool(dev(V, dtype), [dev(a) for a, _, _ in lay],
                                           [dev(b) for _, b, _ in lay],
                                           [dev(c, dtype) for _, _, c in lay])
    ref = np.zeros((N, dv))
    touched = np.zeros(N, bool)
    for l, (idx, w, dy) in enumerate(lay):
        r, d, dw = obag.embbag_bwd(V, idx, w, dy)
        ref[r] += d
        touched[r] = True
        assert_close(host(dws[l]), dw, TOL["f32"], f"dw layer {l}")
    u = int(U.item())
    assert np.array_equal(host(rows[:u]), np.nonzero(touched)[0])      # one row per pooled row
    assert_close(host(dV[:u]), ref[touched], TOL["f32"], "pooled dV")


def test_sparse_adam_matches_oracle():
    from paper_2412_09764_b200 import ops
    N, dv, T, B = 1024, 128, 40, 16
    V = gen.tensor(3, "V", (N, dv), dtype="f32").astype(np.float64)
    Vg = dev(V.astype(np.float32))
    m_g = torch.zeros((N, dv), device="cuda")
    v_g = torch.zeros((N, dv), device="cuda")
    st_g = torch.zeros(N, dtype=torch.int32, device="cuda")
    m, v, st = np.zeros((N, dv)), np.zeros((N, dv)), np.zeros(N, np.int64)
    hp = dict(lr=0.01, beta1=0.9, beta2=0.99, eps=1e-6, weight_decay=0.01)
    for step in range(3):
        idx = streams.zipf_indices(30 + step, T, B, N, 1.0)
        w = streams.softmax_free_weights(30 + step, T, B)
        dy = gen.tensor(30 + step, "dout", (T, dv))
        rows, dV, U, dw = ops.embbag_bwd(Vg, dev(idx), dev(w), dev(dy), sync=False)
        ops.sparse_adam(Vg, rows, dV, U, m_g, v_g, st_g, **hp)
        r, d, _ = obag.embbag_bwd(V, idx, w, dy)   # gradient at the oracle's current V
        ooptim.sparse_adam_step(V, m, v, st, r, d, **hp)
    torch.cuda.synchronize()
    assert np.array_equal(host(st_g), st)
    assert_close(host(m_g), m, TOL["f32"], "m")
    assert_close(host(v_g), v, TOL["f32"], "v")
    assert_close(host(Vg), V, TOL["f32"], "V")
