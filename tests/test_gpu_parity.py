"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element
by element on the same seeded inputs, at sizes spanning several tiles with
ragged tails.  Bit-exact for indices / row sets and for the exact input
classes; otherwise within the north_star tolerances (tests/gpu_util.TOL)."""
import numpy as np
import pytest
import torch

from oracle import bag as obag, layer as olayer, pkm as opkm
from synthetic import gen, streams
from tests.gpu_util import TOL, assert_close, compare_topk, dev, host, layer_magnitudes

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


# ------------------------------------------------------------------ synth
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("cls", [gen.CLS_CONTINUOUS, gen.CLS_EXACT, gen.CLS_DYADIC])
def test_synth_generator_matches_numpy(dtype, cls):
    scale = gen.scale_for("K1", Dk=1024) if cls == gen.CLS_CONTINUOUS else 0.5
    rows, cols, row0 = 37, 48, 1000
    t = torch.empty((rows, cols), dtype=torch.bfloat16 if dtype == "bf16" else torch.float32,
                    device="cuda")
    ops().synth_fill(t, seed=11, tag=gen.TAGS["K1"], scale=scale, cls=cls, row0=row0)
    ref = gen.rows(11, "K1", np.arange(row0, row0 + rows), cols, scale=scale, dtype=dtype, cls=cls)
    assert np.array_equal(t.float().cpu().numpy(), ref)


def test_synth_indices_match_numpy():
    t = torch.empty((64, 128), dtype=torch.int32, device="cuda")
    ops().synth_fill(t, seed=3, tag=gen.TAGS["idx"], cls=3, modulus=1 << 20)
    assert np.array_equal(t.cpu().numpy(), streams.uniform_indices(3, 64, 128, 1 << 20))


# ------------------------------------------------------------ bag forward
BAG_CASES = [  # (dtype, N, dv, T, B)
    ("f32", 1024, 64, 37, 4),
    ("f32", 4096, 128, 129, 16),
    ("bf16", 4096, 256, 67, 128),
    ("bf16", 8192, 2048, 45, 128),
    ("bf16", 2048, 4096, 19, 40),     # two column slices
    ("bf16", 1024, 512, 300, 8),
]


@pytest.mark.parametrize("dtype,N,dv,T,B", BAG_CASES)
def test_embbag_fwd_exact_class_bit_exact(dtype, N, dv, T, B):
    V = gen.tensor(1, "V", (N, dv), dtype=dtype, cls=gen.CLS_EXACT)
    idx = streams.uniform_indices(1, T, B, N)
    w = streams.softmax_free_weights(1, T, B, cls=gen.CLS_DYADIC)
    y = ops().embbag_fwd(dev(V, dtype), dev(idx), dev(w))
    ref = obag.embbag_fwd(V, idx, w)
    # dyadic * exact values: every partial sum is exact in fp32 while
    # |partial| < 2^24/64; the bf16 output rounding is the only error
    want = gen.round_bf16(ref.astype(np.float32)) if dtype == "bf16" else ref
    assert np.array_equal(host(y), want)


@pytest.mark.parametrize("dtype,N,dv,T,B", BAG_CASES)
def test_embbag_fwd_continuous_and_gate(dtype, N, dv, T, B):
    V = gen.tensor(2, "V", (N, dv), dtype=dtype)
    idx = streams.zipf_indices(2, T, B, N, 1.1)
    w = streams.softmax_free_weights(2, T, B)
    g = gen.tensor(2, "x", (T, dv), dtype=dtype) * 3
    g = gen.round_bf16(g) if dtype == "bf16" else g
    z, y = ops().embbag_fwd(dev(V, dtype), dev(idx), dev(w), gate_pre=dev(g, dtype),
                            return_ungated=True)
    ref = obag.embbag_fwd(V, idx, w)
    from oracle.gate import silu
    assert_close(host(y), ref, TOL[dtype], "y")
    assert_close(host(z), ref * silu(g.astype(np.float64)), TOL[dtype], "y*silu(g)")


def test_embbag_fwd_edge_cases():
    o = ops()
    V = gen.tensor(3, "V", (64, 32), dtype="f32")
    # k=1, w=1 -> row copy; w=0 -> 0
    idx = np.array([[5], [63], [0]], np.int32)
    y = o.embbag_fwd(dev(V), dev(idx), dev(np.ones((3, 1), np.float32)))
    assert np.array_equal(host(y), V[[5, 63, 0]])
    y0 = o.embbag_fwd(dev(V), dev(idx), dev(np.zeros((3, 1), np.float32)))
    assert np.all(host(y0) == 0)
    # empty batch is a no-op
    ye = o.embbag_fwd(dev(V), dev(np.zeros((0, 4), np.int32)), dev(np.zeros((0, 4), np.float32)))
    assert ye.shape == (0, 32)


# ----------------------------------------------------------- bag backward
@pytest.mark.parametrize("profile", ["u", "c0", "c50", "c100", "zipf"])
@pytest.mark.parametrize("dtype,dv", [("f32", 64), ("bf16", 2048)])
def test_embbag_bwd_profiles(profile, dtype, dv):
    N, T, B = 1 << 14, 40, 32
    if profile == "u":
        idx = streams.uniform_indices(4, T, B, N)
    elif profile == "zipf":
        idx = streams.zipf_indices(4, T, B, N, 1.1)
    else:
        idx = streams.collision_indices(4, T, B, N, int(profile[1:]))
    V = gen.tensor(4, "V", (N, dv), dtype=dtype, cls=gen.CLS_EXACT)
    w = streams.softmax_free_weights(4, T, B, cls=gen.CLS_DYADIC)
    dy = gen.tensor(4, "dout", (T, dv), dtype=dtype, cls=gen.CLS_EXACT)
    rows, dV, dw = ops().embbag_bwd(dev(V, dtype), dev(idx), dev(w), dev(dy, dtype))
    rr, rdV, rdw = obag.embbag_bwd(V, idx, w, dy)
    assert np.array_equal(host(rows), rr)              # rows = distinct indices
    assert np.array_equal(host(dV), rdV)               # exact class: bit-exact
    assert np.array_equal(host(dw), rdw)


@pytest.mark.parametrize("dtype,dv", [("f32", 64), ("bf16", 256), ("bf16", 4096)])
def test_embbag_bwd_continuous_and_deterministic(dtype, dv):
    N, T, B = 1 << 12, 97, 48
    idx = streams.zipf_indices(5, T, B, N, 0.8)
    V = gen.tensor(5, "V", (N, dv), dtype=dtype)
    w = streams.softmax_free_weights(5, T, B)
    dy = gen.tensor(5, "dout", (T, dv), dtype=dtype)
    a = ops().embbag_bwd(dev(V, dtype), dev(idx), dev(w), dev(dy, dtype))
    b = ops().embbag_bwd(dev(V, dtype), dev(idx), dev(w), dev(dy, dtype))
    for x, y in zip(a, b):                              # determinism
        assert torch.equal(x, y)
    rr, rdV, rdw = obag.embbag_bwd(V, idx, w, dy)
    assert np.array_equal(host(a[0]), rr)
    assert_close(host(a[1]), rdV, TOL["f32"], "dV")     # fp32 accumulation of dtype inputs
    assert_close(host(a[2]), rdw, TOL["f32"], "dw")


@pytest.mark.parametrize("dtype,dv", [("f32", 64), ("bf16", 1024), ("bf16", 2048), ("bf16", 4096)])
def test_embbag_bwd_long_runs_and_grad_apply(dtype, dv):
    """A hot row hit by ~2600 positions: split into 32-position pieces and
    combined in piece order (two-level, counters), for every segmented-kernel
    configuration (one CTA per chunk; pipelined 16- and 32-byte threads; two
    column slices); dense apply equals A^T dy."""
    o = ops()
    N, T, B = 256, 300, 10
    idx = np.full((T, B), 7, np.int32)
    idx.flat[::7] = (np.arange(0, T * B, 7) * 13) % N
    V = gen.tensor(6, "V", (N, dv), dtype=dtype)
    w = streams.softmax_free_weights(6, T, B)
    dy = gen.tensor(6, "dout", (T, dv), dtype=dtype)
    rows, dV, U, dw = o.embbag_bwd(dev(V, dtype), dev(idx), dev(w), dev(dy, dtype), sync=False)
    rr, rdV, rdw = obag.embbag_bwd(V, idx, w, dy)
    u = int(U.item())
    assert np.array_equal(host(rows[:u]), rr)
    assert_close(host(dV[:u]), rdV, TOL["f32"], "dV")
    assert_close(host(dw), rdw, TOL["f32"], "dw")
    if dtype != "f32":
        return
    dense = torch.zeros((N, dv), dtype=torch.float32, device="cuda")
    o.embbag_grad_apply(dev(V), dev(idx), rows, dV, U, dense)
    A = obag.dense_selection_matrix(idx, w, N)
    assert_close(host(dense), A.T @ dy, TOL["f32"], "dense dV")


# ------------------------------------------------------------ product keys
def _pkm_inputs(seed, T, H, S, Dk, dtype, cls):
    sc = gen.scale_for("K1", Dk=Dk) if cls == gen.CLS_CONTINUOUS else 1.0
    q = gen.tensor(seed, "q", (T, H, Dk), dtype=dtype, cls=cls)
    K1 = gen.tensor(seed, "K1", (H, S, Dk // 2), scale=sc, dtype=dtype, cls=cls)
    K2 = gen.tensor(seed, "K2", (H, S, Dk // 2), scale=sc, dtype=dtype, cls=cls)
    return q, K1, K2


PKM_CASES = [  # (dtype, T, H, S, Dk, k)
    ("f32", 256, 1, 32, 32, 4),        # C1 (tiny PKM)
    ("f32", 77, 2, 32, 64, 4),
    ("bf16", 130, 4, 64, 128, 8),
    ("bf16", 70, 4, 128, 256, 32),
    ("bf16", 33, 2, 1024, 1024, 32),   # C2 per-head shapes, few tokens
]


@pytest.mark.parametrize("dtype,T,H,S,Dk,k", PKM_CASES)
def test_pkm_topk_exact_class(dtype, T, H, S, Dk, k):
    """Exact class: scores exact in fp32, so indices AND scores bit-exact with
    the plain definition (brute force over all N = S^2 keys), including the
    many exact ties (tie-break)."""
    q, K1, K2 = _pkm_inputs(8, T, H, S, Dk, dtype, gen.CLS_EXACT)
    idx, w, score = ops().pkm_topk(dev(q, dtype), dev(K1, dtype), dev(K2, dtype), k, with_score=True)
    method = "full" if S * S <= 1 << 14 else "two_stage"
    ridx, rscore, rw = opkm.pkm_lookup(q.astype(np.float64), K1.astype(np.float64),
                                       K2.astype(np.float64), k, method=method)
    assert np.array_equal(host(idx), ridx)
    assert np.array_equal(host(score), rscore)
    assert_close(host(w), rw, 1e-6, "w")
    np.testing.assert_allclose(host(w).sum(-1), 1.0, atol=1e-6)


@pytest.mark.parametrize("dtype,T,H,S,Dk,k", PKM_CASES)
def test_pkm_topk_continuous(dtype, T, H, S, Dk, k):
    q, K1, K2 = _pkm_inputs(9, T, H, S, Dk, dtype, gen.CLS_CONTINUOUS)
    idx, w, score = ops().pkm_topk(dev(q, dtype), dev(K1, dtype), dev(K2, dtype), k, with_score=True)
    q64, K164, K264 = (a.astype(np.float64) for a in (q, K1, K2))
    ridx, rscore, rw = opkm.pkm_lookup(q64, K164, K264, k)
    near = compare_topk(host(idx), ridx, q64, K164, K264)
    ok = np.ones(ridx.shape[:2], bool)
    for t, h, _ in near:
        ok[t, h] = False
    assert_close(host(score)[ok], rscore[ok], 1e-5, "score")
    assert_close(host(w)[ok], rw[ok], TOL["f32"], "w")
    np.testing.assert_allclose(host(w).sum(-1), 1.0, atol=1e-5)


def test_pkm_topk_degenerate_queries():
    """q = 0 -> flat indices 0..k-1, w = 1/k; k = 1 -> w = 1."""
    T, H, S, Dk, k = 5, 2, 32, 32, 6
    _, K1, K2 = _pkm_inputs(10, T, H, S, Dk, "f32", gen.CLS_CONTINUOUS)
    idx, w = ops().pkm_topk(dev(np.zeros((T, H, Dk), np.float32)), dev(K1), dev(K2), k)
    assert np.array_equal(host(idx), np.broadcast_to(np.arange(k), (T, H, k)))
    np.testing.assert_allclose(host(w), 1.0 / k, rtol=1e-6)
    q, _, _ = _pkm_inputs(10, T, H, S, Dk, "f32", gen.CLS_CONTINUOUS)
    idx1, w1 = ops().pkm_topk(dev(q), dev(K1), dev(K2), 1)
    assert np.all(host(w1) == 1.0)


@pytest.mark.parametrize("dtype,T,H,S,Dk,k", PKM_CASES[:4])
def test_pkm_topk_bwd(dtype, T, H, S, Dk, k):
    q, K1, K2 = _pkm_inputs(11, T, H, S, Dk, dtype, gen.CLS_CONTINUOUS)
    q64, K164, K264 = (a.astype(np.float64) for a in (q, K1, K2))
    ridx, rscore, rw = opkm.pkm_lookup(q64, K164, K264, k)
    dw = gen.tensor(11, "dout", (T, H, k), dtype="f32")
    # the backward takes the selection as an input: feed the oracle's
    rdq, rdK1, rdK2, _ = opkm.pkm_bwd(q64, K164, K264, ridx, rw, dw)
    dq, dK1, dK2 = ops().pkm_topk_bwd(dev(q, dtype), dev(K1, dtype), dev(K2, dtype),
                                      dev(ridx.astype(np.int32)), dev(rw.astype(np.float32)), dev(dw))
    # bf16: the dense path rounds the selected score gradients to bf16 before
    # the tensor-core products; fp32 inputs stay fp32 end to end
    tol = TOL[dtype]
    assert_close(host(dq), rdq, tol, "dq")
    assert_close(host(dK1), rdK1, tol, "dK1")
    assert_close(host(dK2), rdK2, tol, "dK2")


# ------------------------------------------------------------ memory layer
LAYER_CASES = [  # (dtype, T, H, S, Dk, k, dv, D, gated)
    ("f32", 256, 1, 32, 32, 4, 64, 64, True),      # C1
    ("f32", 256, 1, 32, 64, 4, 64, 64, False),     # C1, Dk = 64, vanilla Memory
    ("f32", 99, 2, 32, 32, 4, 128, 64, True),
    ("bf16", 150, 4, 64, 128, 8, 256, 256, True),
    ("bf16", 64, 4, 128, 512, 32, 1024, 512, True),
]


@pytest.mark.parametrize("dtype,T,H,S,Dk,k,dv,D,gated", LAYER_CASES)
def test_memory_layer_fwd_bwd(dtype, T, H, S, Dk, k, dv, D, gated):
    seed = 12
    f = lambda tag, shape, sc=1.0: gen.tensor(seed, tag, shape, scale=sc, dtype=dtype)
    h = dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)),
             K1=f("K1", (H, S, Dk // 2), gen.scale_for("K1", Dk=Dk)),
             K2=f("K2", (H, S, Dk // 2), gen.scale_for("K2", Dk=Dk)),
             V=f("V", (S * S, dv)), W1=f("W1", (D, dv), gen.scale_for("W1", D=D)),
             W2=f("W2", (dv, D), gen.scale_for("W2", dv=dv)),
             dout=f("dout", (T, D if gated else dv)))
    t = {n: dev(a, dtype) for n, a in h.items()}
    o = ops()
    out, saved = o.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"],
                                    k, gated=gated)
    g = o.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"],
                           saved, want_dw=True)
    h64 = {n: a.astype(np.float64) for n, a in h.items()}
    rout, rs = olayer.memory_layer_fwd(h64["x"], h64["q"], h64["K1"], h64["K2"], h64["V"],
                                       h64["W1"], h64["W2"], k, gated=gated)
    near = compare_topk(host(saved["idx"]), rs["idx"], h64["q"], h64["K1"], h64["K2"])
    assert not near, f"near ties in a small case: {near}"
    r = olayer.memory_layer_bwd(h64["dout"], h64["x"], h64["q"], h64["K1"], h64["K2"], h64["V"],
                                h64["W1"], h64["W2"], rs, gated=gated)
    tol = TOL[dtype]
    # bf16: elementwise rounding-model bound on top of Q17
    m = layer_magnitudes(h64, rs, r, gated) if dtype == "bf16" else {}
    assert_close(host(out), rout, tol, "out", mag=m.get("out"))
    U = int(g["U"].item())
    assert np.array_equal(host(g["rows"][:U]), r["rows"])
    for n in ("dV", "dw", "dq", "dK1", "dK2") + (("dx", "dW1", "dW2") if gated else ()):
        got = host(g[n][:U]) if n == "dV" else host(g[n])
        assert_close(got, r[n], tol, n, mag=m.get(n))


@pytest.mark.parametrize("dtype,T,H,S,Dk,k,dv,D,gated", [LAYER_CASES[0], LAYER_CASES[3]])
def test_memory_layer_state_path_bit_identical(dtype, T, H, S, Dk, k, dv, D, gated):
    """memory_layer_fwd_state / memory_layer_bwd_state (inverse map built by
    the forward on a side stream) == the plain pair, bit for bit."""
    seed = 13
    f = lambda tag, shape, sc=1.0: gen.tensor(seed, tag, shape, scale=sc, dtype=dtype)
    h = dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)),
             K1=f("K1", (H, S, Dk // 2), gen.scale_for("K1", Dk=Dk)),
             K2=f("K2", (H, S, Dk // 2), gen.scale_for("K2", Dk=Dk)),
             V=f("V", (S * S, dv)), W1=f("W1", (D, dv), gen.scale_for("W1", D=D)),
             W2=f("W2", (dv, D), gen.scale_for("W2", dv=dv)), dout=f("dout", (T, D)))
    t = {n: dev(a, dtype) for n, a in h.items()}
    o = ops()
    res = []
    for keep in (False, True):
        out, saved = o.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                                        t["W2"], k, gated=gated, keep_state=keep)
        assert (saved["state"] is not None) == keep
        g = o.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                               t["W2"], saved, want_dw=True)
        U = int(g["U"].item())
        res.append(dict(out=host(out), U=U, rows=host(g["rows"][:U]), dV=host(g["dV"][:U]),
                        dw=host(g["dw"]), dq=host(g["dq"]), dK1=host(g["dK1"]), dx=host(g["dx"])))
    a, b = res
    for n in a:
        assert np.array_equal(a[n], b[n]), n


@pytest.mark.parametrize("dtype,dv", [("f32", 64), ("bf16", 256), ("bf16", 2048)])
def test_embbag_bwd_prepared_state_bit_identical(dtype, dv):
    """embbag_bwd_prepare + embbag_bwd(state=) == embbag_bwd, bit for bit."""
    N, T, B = 4096, 300, 64
    idx = streams.uniform_indices(3, T, B, N)
    w = gen.tensor(3, "w", (T, B)).astype(np.float32)
    dy = gen.tensor(3, "dout", (T, dv), dtype=dtype)
    V = gen.tensor(3, "V", (N, dv), dtype=dtype)
    o = ops()
    Vd, idd, wd, dyd = dev(V, dtype), dev(idx), dev(w), dev(dy, dtype)
    a = o.embbag_bwd(Vd, idd, wd, dyd)
    st = o.embbag_bwd_prepare(N, dv, idd, Vd.dtype)
    b = o.embbag_bwd(Vd, idd, wd, dyd, state=st)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


@pytest.mark.parametrize("keep_state", [False, True])
def test_memory_layer_deterministic(keep_state):
    """SURVEY §8 determinism pin: two runs give bitwise-equal idx / w / out /
    dV / dw / dq / dK / dx / dW (sorted segments, fixed orders, no atomics)."""
    dtype, T, H, S, Dk, k, dv, D = "bf16", 150, 4, 64, 128, 8, 256, 256
    seed = 14
    f = lambda tag, shape, sc=1.0: gen.tensor(seed, tag, shape, scale=sc, dtype=dtype)
    h = dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)),
             K1=f("K1", (H, S, Dk // 2), gen.scale_for("K1", Dk=Dk)),
             K2=f("K2", (H, S, Dk // 2), gen.scale_for("K2", Dk=Dk)),
             V=f("V", (S * S, dv)), W1=f("W1", (D, dv), gen.scale_for("W1", D=D)),
             W2=f("W2", (dv, D), gen.scale_for("W2", dv=dv)), dout=f("dout", (T, D)))
    t = {n: dev(a, dtype) for n, a in h.items()}
    o = ops()
    runs = []
    for _ in range(2):
        out, saved = o.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"],
                                        k, keep_state=keep_state)
        g = o.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                               t["W2"], saved, want_dw=True)
        U = int(g["U"].item())
        runs.append([out, saved["idx"], saved["w"], g["rows"][:U], g["dV"][:U], g["dw"], g["dq"],
                     g["dK1"], g["dK2"], g["dx"], g["dW1"], g["dW2"]])
    for a, b in zip(*runs):
        assert torch.equal(a, b)


# ------------------------------------------------------------ edge cases
def test_out_of_range_index_reported_under_check_mode():
    """S:233 index error: with ML_CHECK_INDICES=1 an index >= N is reported
    as ML_ERR_INDEX (clamped to row 0 / weight 0 on the device, no fault)."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import numpy as np, torch
        from paper_2412_09764_b200 import ops, MemlayerError
        V = torch.ones((64, 32), device="cuda")
        idx = torch.tensor([[1, 2], [3, 64]], dtype=torch.int32, device="cuda")
        w = torch.ones((2, 2), device="cuda")
        try:
            ops.embbag_fwd(V, idx, w)
            print("NO_ERROR")
        except MemlayerError as e:
            print("STATUS", e.status)
        idx[1, 1] = 5
        y = ops.embbag_fwd(V, idx, w)
        print("OK_AFTER", float(y.sum()))
    """)
    env = dict(__import__("os").environ, ML_CHECK_INDICES="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=300)
    assert "STATUS 3" in r.stdout, r.stdout + r.stderr
    assert "OK_AFTER 128.0" in r.stdout, r.stdout + r.stderr


def test_empty_batches():
    o = ops()
    V = torch.ones((64, 32), device="cuda")
    idx = torch.zeros((0, 4), dtype=torch.int32, device="cuda")
    w = torch.zeros((0, 4), device="cuda")
    rows, dV, U, dw = o.embbag_bwd(V, idx, w, torch.zeros((0, 32), device="cuda"), sync=False)
    assert int(U.item()) == 0 and dw.shape == (0, 4)
    q = torch.zeros((0, 1, 32), device="cuda")
    K = torch.zeros((1, 32, 16), device="cuda")
    i2, w2 = o.pkm_topk(q, K, K, 4)
    assert i2.shape == (0, 1, 4)


def test_k_equals_S_and_k1_layer_corner():
    """k = S (every half key selected) and k = 1 (w = 1, dq = dK = 0)."""
    o = ops()
    T, H, S, Dk = 40, 2, 32, 32
    q, K1, K2 = _pkm_inputs(13, T, H, S, Dk, "f32", gen.CLS_CONTINUOUS)
    q64, K164, K264 = (a.astype(np.float64) for a in (q, K1, K2))
    idx, w = o.pkm_topk(dev(q), dev(K1), dev(K2), 32)
    ridx, _, rw = opkm.pkm_lookup(q64, K164, K264, 32)
    compare_topk(host(idx), ridx, q64, K164, K264)
    idx1, w1 = o.pkm_topk(dev(q), dev(K1), dev(K2), 1)
    dq, dK1, dK2 = o.pkm_topk_bwd(dev(q), dev(K1), dev(K2), idx1, w1,
                                  dev(gen.tensor(13, "dout", (T, H, 1))))
    assert torch.all(dq == 0) and torch.all(dK1 == 0) and torch.all(dK2 == 0)


# ------------------------------------------ backward strategy controls (f3)
@pytest.mark.parametrize("profile", ["u", "c50", "zipf"])
@pytest.mark.parametrize("dtype,dv", [("f32", 64), ("bf16", 256), ("bf16", 2048), ("bf16", 4096)])
def test_backward_strategies_agree(profile, dtype, dv):
    """"atomics" and "lock" agree with the sequential scatter-add
    oracle within fp32 reordering (rel 1e-5 of the row scale); the sorted
    "reverse_indices" value gradient equals it on the exact class bit for bit."""
    o = ops()
    N, T, B = 1 << 12, 64, 32
    idx = {"u": streams.uniform_indices(7, T, B, N), "zipf": streams.zipf_indices(7, T, B, N, 1.1),
           "c50": streams.collision_indices(7, T, B, N, 50)}[profile]
    w = streams.softmax_free_weights(7, T, B)
    dy = gen.tensor(7, "dout", (T, dv), dtype=dtype)
    A = obag.dense_selection_matrix(idx, w, N)
    ref = A.T @ dy.astype(np.float64)
    # rigorous fp32 summation bound of an arbitrary-order sum of n terms:
    # |err| <= (n - 1) 2^-24 sum|terms| (+ one rounding per product)
    n_r = np.bincount(idx.reshape(-1), minlength=N)[:, None]
    bound = (n_r + 1) * 2.0 ** -24 * (np.abs(A).T @ np.abs(dy.astype(np.float64)))
    da = o.embbag_bwd_atomics(N, dev(idx), dev(w), dev(dy, dtype))
    dl = o.embbag_bwd_lock(N, dev(idx), dev(w), dev(dy, dtype))
    for name, got in (("atomics", host(da)), ("lock", host(dl))):
        err = np.abs(got - ref)
        assert np.all(err <= bound + 1e-12), (name, float((err - bound).max()))
        assert err.max() <= 1e-5 * np.abs(ref).max(), name
    rows, dV = o.embbag_bwd_dv_only(N, dev(idx), dev(w), dev(dy, dtype))
    assert np.array_equal(host(rows), np.unique(idx))
    assert_close(host(dV), ref[np.unique(idx)], 1e-5, "reverse_indices")


# ------------------------------------------------------------ qk-norm (f2)
@pytest.mark.parametrize("dtype,T,H,S,Dk,k", [("f32", 77, 2, 32, 64, 4), ("bf16", 70, 4, 128, 256, 32)])
def test_pkm_topk_qk_norm(dtype, T, H, S, Dk, k):
    q, K1, K2 = _pkm_inputs(14, T, H, S, Dk, dtype, gen.CLS_CONTINUOUS)
    q64, K164, K264 = (a.astype(np.float64) for a in (q, K1, K2))
    idx, w, score = ops().pkm_topk(dev(q, dtype), dev(K1, dtype), dev(K2, dtype), k,
                                   with_score=True, qk_norm=True)
    ridx, rscore, rw = opkm.pkm_lookup(q64, K164, K264, k, qk_norm=True)
    qn, K1n, K2n = opkm._qk(q64, K164, K264)
    near = compare_topk(host(idx), ridx, qn, K1n, K2n)
    ok = np.ones(ridx.shape[:2], bool)
    for t, h, _ in near:
        ok[t, h] = False
    assert np.abs(host(score)).max() <= 2.0 + 1e-5            # two normalised halves
    assert_close(host(score)[ok], rscore[ok], 1e-5, "score")
    assert_close(host(w)[ok], rw[ok], TOL["f32"], "w")
    dw = gen.tensor(14, "dout", (T, H, k), dtype="f32")
    rdq, rdK1, rdK2, _ = opkm.pkm_bwd(q64, K164, K264, ridx, rw, dw, qk_norm=True)
    dq, dK1, dK2 = ops().pkm_topk_bwd(dev(q, dtype), dev(K1, dtype), dev(K2, dtype),
                                      dev(ridx.astype(np.int32)), dev(rw.astype(np.float32)),
                                      dev(dw), qk_norm=True)
    assert_close(host(dq), rdq, TOL[dtype], "dq")
    assert_close(host(dK1), rdK1, TOL[dtype], "dK1")
    assert_close(host(dK2), rdK2, TOL[dtype], "dK2")


@pytest.mark.parametrize("dtype,T,H,S,Dk,k,dv,D", [("f32", 128, 1, 32, 32, 4, 64, 64),
                                                  ("bf16", 96, 4, 64, 128, 8, 256, 256)])
def test_memory_layer_qk_norm(dtype, T, H, S, Dk, k, dv, D):
    seed = 15
    f = lambda tag, shape, sc=1.0: gen.tensor(seed, tag, shape, scale=sc, dtype=dtype)
    h = dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)), K1=f("K1", (H, S, Dk // 2)),
             K2=f("K2", (H, S, Dk // 2)), V=f("V", (S * S, dv)),
             W1=f("W1", (D, dv), gen.scale_for("W1", D=D)), W2=f("W2", (dv, D), gen.scale_for("W2", dv=dv)),
             dout=f("dout", (T, D)))
    t = {n: dev(a, dtype) for n, a in h.items()}
    o = ops()
    out, saved = o.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"], k,
                                    qk_norm=True)
    g = o.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"], saved)
    h64 = {n: a.astype(np.float64) for n, a in h.items()}
    rout, rs = olayer.memory_layer_fwd(h64["x"], h64["q"], h64["K1"], h64["K2"], h64["V"], h64["W1"],
                                       h64["W2"], k, qk_norm=True)
    qn, K1n, K2n = opkm._qk(h64["q"], h64["K1"], h64["K2"])
    assert not compare_topk(host(saved["idx"]), rs["idx"], qn, K1n, K2n)
    r = olayer.memory_layer_bwd(h64["dout"], h64["x"], h64["q"], h64["K1"], h64["K2"], h64["V"],
                                h64["W1"], h64["W2"], rs)
    tol = TOL[dtype]
    m = {}
    if dtype == "bf16":
        # magnitudes on the normalised operands; the normalisation's backward
        # (I - x^ x^T) / |x| at most doubles them, scaled by the inverse norms
        hn = dict(h64, q=qn, K1=K1n, K2=K2n)
        m = layer_magnitudes(hn, rs, r)
        Dh = Dk // 2
        qh = h64["q"].reshape(T, H, 2, Dh)
        qinv = 1.0 / np.maximum(np.linalg.norm(qh, axis=-1), 1e-6)
        m["dq"] = (m["dq"].reshape(T, H, 2, Dh) * 2 * qinv[..., None]).reshape(T, H, Dk)
        for n, K in (("dK1", h64["K1"]), ("dK2", h64["K2"])):
            m[n] = m[n] * 2 / np.maximum(np.linalg.norm(K, axis=-1, keepdims=True), 1e-6)
    assert_close(host(out), rout, tol, "out", mag=m.get("out"))
    assert_close(host(g["dq"]), r["dq"], tol, "dq", mag=m.get("dq"))
    assert_close(host(g["dK1"]), r["dK1"], tol, "dK1", mag=m.get("dK1"))
    assert_close(host(g["dK2"]), r["dK2"], tol, "dK2", mag=m.get("dK2"))


@pytest.mark.slow
def test_embbag_bwd_large_position_count():
    """8.4M positions (the 4-/8-way group's per-rank size): the single-pass
    run kernels and the look-back sort; rows are the distinct indices and
    sampled rows' dV equal their oracle sums (Zipf stream: long runs too)."""
    o = ops()
    N, dv, T, B = 1 << 20, 64, 65536, 128
    idx = streams.zipf_indices(15, T, B, N, 0.8)
    w = streams.softmax_free_weights(15, T, B)
    dy = gen.tensor(15, "dout", (T, dv), dtype="f32")
    V = gen.tensor(15, "V", (N, dv), dtype="f32")
    rows, dV, U, dw = o.embbag_bwd(dev(V), dev(idx), dev(w), dev(dy), sync=False)
    u = int(U.item())
    flat = idx.reshape(-1)
    ur = np.unique(flat)
    assert u == ur.size and np.array_equal(host(rows[:u]), ur)
    rng = np.random.default_rng(0)
    order = np.argsort(flat, kind="stable")
    starts = np.searchsorted(flat[order], ur)
    ends = np.searchsorted(flat[order], ur, side="right")
    pick = np.concatenate([np.argsort(ends - starts)[-8:], rng.choice(ur.size, 56, replace=False)])
    gdV = host(dV[:u])
    for j in pick:
        pos = order[starts[j]:ends[j]]
        ref = (w.reshape(-1)[pos, None].astype(np.float64) * dy[pos // B].astype(np.float64)).sum(0)
        assert_close(gdV[j], ref, TOL["f32"], f"dV[{ur[j]}]")
    sp = rng.choice(T * B, 256, replace=False)
    refdw = np.einsum("pd,pd->p", dy[sp // B].astype(np.float64), V[flat[sp]].astype(np.float64))
    assert_close(host(dw).reshape(-1)[sp], refdw, TOL["f32"], "dw")


def test_out_of_range_index_backward_row0_weight0():
    """ADVICE r1 / memlayer.h: an index outside [0, N) is clamped to row 0 with
    weight 0 in the backward as in the forward -- for N not a power of two
    too (N = 1000, index 1010 < 2^10): no row >= N, no value row read past the
    end, and dV[0] receives nothing from the clamped positions (dw of a
    clamped position is <dy, V[0]>, the gradient of its weight at row 0)."""
    o = ops()
    N, dv, T, B = 1000, 256, 40, 16
    V = gen.tensor(21, "V", (N, dv), dtype="f32")
    idx = streams.uniform_indices(21, T, B, N)
    w = streams.softmax_free_weights(21, T, B)
    dy = gen.tensor(21, "dout", (T, dv), dtype="f32")
    bad = [(0, 3, 1010), (5, 0, 1023), (7, 9, 5000), (11, 2, -3)]
    for t, j, v in bad:
        idx[t, j] = v
    rows, dV, U, dw = o.embbag_bwd(dev(V), dev(idx), dev(w), dev(dy), sync=False)
    torch.cuda.synchronize()
    ie, we = idx.copy(), w.copy()
    for t, j, _ in bad:
        ie[t, j], we[t, j] = 0, 0.0
    rr, rdV, rdw = obag.embbag_bwd(V, ie, we, dy)
    u = int(U.item())
    assert np.array_equal(host(rows[:u]), rr) and rr.max() < N
    assert_close(host(dV[:u]), rdV, TOL["f32"], "dV")
    assert_close(host(dw), rdw, TOL["f32"], "dw")
    y = o.embbag_fwd(dev(V), dev(idx), dev(w))
    assert_close(host(y), obag.embbag_fwd(V, ie, we), TOL["f32"], "y")


@pytest.mark.parametrize("N,dv,T,B", [(4096, 256, 300, 64), (1 << 16, 2048, 150, 128),
                                      (8192, 4096, 40, 128), (2000, 512, 257, 32)])
def test_bf16_value_gradient_is_rounded_fp32(N, dv, T, B):
    """grad_dtype = bf16 (memlayer.h): every dV element is the fp32 sum of the
    fp32 path rounded once to bf16 -> bit-identical to rounding the fp32
    result; rows, U and dw are unchanged.  Covers both segmented kernels
    (row slices < 2 KiB and >= 2 KiB), long runs (Zipf) and the consumers
    (embbag_grad_apply, sparse Adam) of a bf16 dV."""
    o = ops()
    V = gen.tensor(22, "V", (N, dv), dtype="bf16")
    idx = streams.zipf_indices(22, T, B, N, 1.1)
    w = streams.softmax_free_weights(22, T, B)
    dy = gen.tensor(22, "dout", (T, dv), dtype="bf16")
    Vd, idd, wd, dyd = dev(V, "bf16"), dev(idx), dev(w), dev(dy, "bf16")
    r32, d32, U32, w32 = o.embbag_bwd(Vd, idd, wd, dyd, sync=False)
    r16, d16, U16, w16 = o.embbag_bwd(Vd, idd, wd, dyd, sync=False, grad_dtype=torch.bfloat16)
    u = int(U32.item())
    assert int(U16.item()) == u and d16.dtype == torch.bfloat16
    assert torch.equal(r16[:u], r32[:u]) and torch.equal(w16, w32)
    assert torch.equal(d16[:u], d32[:u].to(torch.bfloat16))
    dense32 = torch.zeros((N, dv), dtype=torch.float32, device="cuda")
    dense16 = torch.zeros((N, dv), dtype=torch.float32, device="cuda")
    o.embbag_grad_apply(Vd, idd, r32, d32[:, :].to(torch.bfloat16).contiguous(), U32, dense32)
    o.embbag_grad_apply(Vd, idd, r16, d16, U16, dense16)
    assert torch.equal(dense32, dense16)
