"""GPU parity of the PEER-style workload (reading Q21):
peer_fwd / peer_bwd through the C ABI vs oracle/peer.py on the same seeded
inputs, element by element (tolerances of tests/gpu_util.TOL)."""
import numpy as np
import pytest
import torch

from oracle import peer as opeer
from synthetic import gen
from tests.gpu_util import TOL, assert_close, compare_topk, dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_09764_b200 import ops  # noqa: F401
    yield


CASES = [  # (dtype, T, H, S, Dk, k, D)
    ("f32", 200, 1, 32, 32, 4, 64),
    ("f32", 77, 2, 32, 64, 8, 128),
    ("bf16", 150, 4, 64, 128, 8, 256),
    ("bf16", 64, 4, 128, 512, 32, 1024),
]


@pytest.mark.parametrize("dtype,T,H,S,Dk,k,D,qk_norm", [c + (False,) for c in CASES] +
                         [("bf16", 150, 4, 64, 128, 8, 256, True), ("f32", 77, 2, 32, 64, 8, 128, True)])
def test_peer_fwd_bwd(dtype, T, H, S, Dk, k, D, qk_norm):
    from paper_2412_09764_b200 import ops as o
    seed = 21
    f = lambda tag, shape, sc=1.0: gen.tensor(seed, tag, shape, scale=sc, dtype=dtype)
    h = dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)),
             K1=f("K1", (H, S, Dk // 2), gen.scale_for("K1", Dk=Dk)),
             K2=f("K2", (H, S, Dk // 2), gen.scale_for("K2", Dk=Dk)),
             U=f("W1", (S * S, D), gen.scale_for("W1", D=D)), V=f("V", (S * S, D)),
             dy=f("dout", (T, D)))
    t = {n: dev(a, dtype) for n, a in h.items()}
    y, saved = o.peer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["U"], t["V"], k, qk_norm=qk_norm)
    g = o.peer_bwd(t["dy"], t["x"], t["q"], t["K1"], t["K2"], t["U"], t["V"], saved, want_dwr=True)
    h64 = {n: a.astype(np.float64) for n, a in h.items()}
    ry, rs = opeer.peer_fwd(h64["x"], h64["q"], h64["K1"], h64["K2"], h64["U"], h64["V"], k,
                            qk_norm=qk_norm)
    if qk_norm:   # near-tie rule on the normalised operands
        from oracle import pkm as opkm
        qn, K1n, K2n = opkm._qk(h64["q"], h64["K1"], h64["K2"])
        near = compare_topk(host(saved["idx"]), rs["idx"], qn, K1n, K2n)
    else:
        near = compare_topk(host(saved["idx"]), rs["idx"], h64["q"], h64["K1"], h64["K2"])
    assert not near, f"near ties in a small case: {near}"
    r = opeer.peer_bwd(h64["dy"], h64["x"], h64["q"], h64["K1"], h64["K2"], h64["U"], h64["V"], rs)
    tol = TOL[dtype]
    assert_close(host(saved["h"]), rs["h"].reshape(T, H, k), tol, "h")
    assert_close(host(y), ry, tol, "y")
    U = int(g["U"].item())
    assert np.array_equal(host(g["rows"][:U]), r["rows"])
    assert_close(host(g["dV"][:U]), r["dV"], tol, "dV")
    assert_close(host(g["dU"][:U]), r["dU"], tol, "dU")
    assert_close(host(g["dx"]), r["dx"], tol, "dx")
    assert_close(host(g["dwr"]), r["dwr"], tol, "dwr")
    assert_close(host(g["dq"]), r["dq"], tol, "dq")
    assert_close(host(g["dK1"]), r["dK1"], tol, "dK1")
    assert_close(host(g["dK2"]), r["dK2"], tol, "dK2")
