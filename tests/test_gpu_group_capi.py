"""The memory group through the C ABI (include/memlayer.h memory_layer_*_group,
embbag_*_group; §3.1.2) on one GPU.

* Hub transport: G ranks as host threads, each with its own stream, running
  exactly the library's protocol code (packed (idx, w) all-gather, block-wise
  bag forward + exchange, dy all-to-all, local sorted backward, dw
  reduce-scatter); the collectives are host-synchronised device copies, so no
  kernel waits on another.  Every rank is checked against the fp64 oracle
  (oracle/group.py for the bag outputs, oracle/layer.py for the rest) with
  the rounding-model bound, and against the unsharded CUDA layer bit-exactly
  where the arithmetic is identical (indices, y, dV rows, the dV slice).
* NCCL transport at G = 1 (the only rank count one GPU allows): bit-identical
  to the hub transport at G = 1.
"""
import threading

import numpy as np
import pytest
import torch

from oracle import group as ogroup, layer as olayer
from synthetic import gen
from tests.gpu_util import TOL, assert_close, compare_topk, host, layer_magnitudes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_09764_b200 import ops  # noqa: F401  (fails loudly without the .so)
    yield


def _inputs(seed, T, H, S, Dk, dv, D, dt="bf16"):
    f = lambda tag, shape, sc=1.0: gen.tensor(seed, tag, shape, scale=sc, dtype=dt)
    return dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)),
                K1=f("K1", (H, S, Dk // 2), gen.scale_for("K1", Dk=Dk)),
                K2=f("K2", (H, S, Dk // 2), gen.scale_for("K2", Dk=Dk)),
                V=f("V", (S * S, dv)), W1=f("W1", (D, dv), gen.scale_for("W1", D=D)),
                W2=f("W2", (dv, D), gen.scale_for("W2", dv=dv)), dout=f("dout", (T, D)))


def _run_hub(t, G, T_loc, dv, k, mode, p2p=False):
    from paper_2412_09764_b200 import ops
    hub = ops.group_hub(G)
    res, errs = [None] * G, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            grp = ops.Group.from_hub(hub, r).set_p2p(p2p)
            with torch.cuda.stream(torch.cuda.Stream()):
                sl = slice(r * T_loc, (r + 1) * T_loc)
                lo, hi = r * dv // G, (r + 1) * dv // G
                Vs = t["V"][:, lo:hi].contiguous()
                x, q, dout = (t[n][sl].contiguous() for n in ("x", "q", "dout"))
                out, sv = ops.memory_layer_fwd_group(grp, x, q, t["K1"], t["K2"], Vs, t["W1"],
                                                     t["W2"], k, mode=mode)
                g = ops.memory_layer_bwd_group(grp, dout, x, q, t["K1"], t["K2"], Vs, t["W1"],
                                               t["W2"], sv, want_dw=True)
                torch.cuda.current_stream().synchronize()
                res[r] = (out, sv, g)
            grp.close()
        except Exception as e:  # surface thread failures
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    ops.group_hub_destroy(hub)
    assert not errs, errs
    return res


@pytest.mark.parametrize("G,mode,p2p", [(1, "alltoall", False), (2, "alltoall", False),
                                         (4, "alltoall", False), (1, "allgather", False),
                                         (2, "allgather", False), (4, "allgather", False),
                                         (2, "alltoall", True), (4, "alltoall", True),
                                         (2, "allgather", True)])
def test_capi_group_layer_vs_oracle(G, mode, p2p):
    """p2p: the fused forward exchange (ml_group_set_p2p), the bag kernel of
    every block storing straight into the owner's exchange region."""
    from paper_2412_09764_b200 import ops
    T_loc, H, S, Dk, k, dv, D = 96, 4, 64, 128, 8, 512, 256
    T = G * T_loc
    h = _inputs(5, T, H, S, Dk, dv, D)
    t = {n: torch.from_numpy(a).to(torch.bfloat16).cuda() for n, a in h.items()}
    out_u, saved_u = ops.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                                          t["W2"], k)
    ref_u = ops.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                                 t["W2"], saved_u, want_dw=True)
    U_u = int(ref_u["U"].item())
    res = _run_hub(t, G, T_loc, dv, k, mode, p2p=p2p)

    h64 = {n: a.astype(np.float64) for n, a in h.items()}
    rout, rs = olayer.memory_layer_fwd(h64["x"], h64["q"], h64["K1"], h64["K2"], h64["V"],
                                       h64["W1"], h64["W2"], k)
    assert not compare_topk(host(saved_u["idx"]), rs["idx"], h64["q"], h64["K1"], h64["K2"])
    rb = olayer.memory_layer_bwd(h64["dout"], h64["x"], h64["q"], h64["K1"], h64["K2"], h64["V"],
                                 h64["W1"], h64["W2"], rs)
    m = layer_magnitudes(h64, rs, rb)
    B = H * k
    idx_r = [rs["idx"][r * T_loc:(r + 1) * T_loc].reshape(T_loc, B) for r in range(G)]
    w_r = [rs["w"][r * T_loc:(r + 1) * T_loc].reshape(T_loc, B) for r in range(G)]
    ry = ogroup.group_fwd(h64["V"], idx_r, w_r, G, mode=mode)
    dK1 = sum(host(res[r][2]["dK1"]) for r in range(G))
    dK2 = sum(host(res[r][2]["dK2"]) for r in range(G))
    dW1 = sum(host(res[r][2]["dW1"]) for r in range(G))
    dW2 = sum(host(res[r][2]["dW2"]) for r in range(G))
    for r in range(G):
        o, sv, g = res[r]
        sl = slice(r * T_loc, (r + 1) * T_loc)
        lo, hi = r * dv // G, (r + 1) * dv // G
        # bit-exact where the arithmetic is the unsharded layer's
        assert torch.equal(sv["idx"], saved_u["idx"][sl])
        assert torch.equal(sv["idx_all"], saved_u["idx"]) and torch.equal(sv["w_all"], saved_u["w"])
        assert torch.equal(sv["y"], saved_u["y"][sl])
        if mode == "allgather":
            assert torch.equal(sv["y_all"], saved_u["y"])
        u = int(g["U"].item())
        assert u == U_u and torch.equal(g["rows"][:u], ref_u["rows"][:U_u])
        assert torch.equal(g["dV"][:u], ref_u["dV"][:U_u, lo:hi])
        # every rank against the oracle
        want_y = ry[r] if mode == "alltoall" else ry[r][sl]
        assert_close(host(sv["y"]), want_y, TOL["bf16"], f"y rank {r}", mag=m["y"][sl])
        assert_close(host(o), rout[sl], TOL["bf16"], f"out rank {r}", mag=m["out"][sl])
        assert np.array_equal(host(g["rows"][:u]), rb["rows"])
        assert_close(host(g["dV"][:u]), rb["dV"][:, lo:hi], TOL["bf16"], f"dV shard {r}",
                     mag=m["dV"][:, lo:hi])
        for n in ("dw", "dq", "dx"):
            assert_close(host(g[n]), rb[n][sl], TOL["bf16"], f"{n} rank {r}", mag=m[n][sl])
    for n, got in (("dK1", dK1), ("dK2", dK2), ("dW1", dW1), ("dW2", dW2)):
        assert_close(got, rb[n], TOL["bf16"], f"{n} vs oracle", mag=m[n])


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("mode", ["alltoall", "allgather"])
def test_capi_group_bag_level(G, mode):
    """embbag_fwd_group / embbag_bwd_group: y and dV bit-exact against the
    unsharded bag (each element keeps its accumulation order), dw within the
    fp32 tolerance (re-associated over the shards)."""
    from paper_2412_09764_b200 import ops
    from synthetic import streams
    N, dv, T_loc, B = 4096, 512, 64, 32
    T = G * T_loc
    V = torch.from_numpy(gen.tensor(6, "V", (N, dv), dtype="bf16")).to(torch.bfloat16).cuda()
    idx = torch.from_numpy(streams.zipf_indices(6, T, B, N, 1.1)).cuda()
    w = torch.from_numpy(streams.softmax_free_weights(6, T, B)).cuda()
    dy = torch.from_numpy(gen.tensor(6, "dout", (T, dv), dtype="bf16")).to(torch.bfloat16).cuda()
    y_u = ops.embbag_fwd(V, idx, w)
    rows_u, dV_u, U_u, dw_u = ops.embbag_bwd(V, idx, w, dy, sync=False)
    hub = ops.group_hub(G)
    res, errs = [None] * G, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            grp = ops.Group.from_hub(hub, r)
            with torch.cuda.stream(torch.cuda.Stream()):
                sl = slice(r * T_loc, (r + 1) * T_loc)
                Vs = V[:, r * dv // G:(r + 1) * dv // G].contiguous()
                y, ia, wa = ops.embbag_fwd_group(grp, Vs, idx[sl].contiguous(), w[sl].contiguous(),
                                                 mode=mode)
                d = dy[sl].contiguous() if mode == "alltoall" else dy
                rows, dV, U, dw = ops.embbag_bwd_group(grp, Vs, ia, wa, d, mode=mode)
                torch.cuda.current_stream().synchronize()
                res[r] = (y, ia, wa, rows, dV, U, dw)
            grp.close()
        except Exception as e:
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    ops.group_hub_destroy(hub)
    assert not errs, errs
    u0 = int(U_u.item())
    for r in range(G):
        y, ia, wa, rows, dV, U, dw = res[r]
        sl = slice(r * T_loc, (r + 1) * T_loc)
        assert torch.equal(ia, idx) and torch.equal(wa, w)
        assert torch.equal(y, y_u[sl] if mode == "alltoall" else y_u)
        u = int(U.item())
        assert u == u0 and torch.equal(rows[:u], rows_u[:u0])
        assert torch.equal(dV[:u], dV_u[:u0, r * dv // G:(r + 1) * dv // G])
        assert_close(host(dw), host(dw_u[sl]), TOL["f32"], f"dw rank {r}")


def test_capi_group_nccl_single_rank_equals_hub():
    """ml_group_init (NCCL) with one rank runs the same protocol as the hub
    transport: results bit-identical."""
    import os
    from paper_2412_09764_b200 import ops
    os.environ.setdefault("NCCL_P2P_DISABLE", "0")
    try:
        uid = ops.group_unique_id()
        grp = ops.Group.nccl(uid, 1, 0)
    except Exception as e:  # no NCCL in this process image
        pytest.skip(f"NCCL unavailable: {e}")
    T_loc, H, S, Dk, k, dv, D = 96, 4, 64, 128, 8, 512, 256
    h = _inputs(7, T_loc, H, S, Dk, dv, D)
    t = {n: torch.from_numpy(a).to(torch.bfloat16).cuda() for n, a in h.items()}
    out, sv = ops.memory_layer_fwd_group(grp, t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                                         t["W2"], k)
    g = ops.memory_layer_bwd_group(grp, t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"],
                                   t["W1"], t["W2"], sv, want_dw=True)
    torch.cuda.synchronize()
    grp.close()
    ref = _run_hub(t, 1, T_loc, dv, k, "alltoall")[0]
    assert torch.equal(out, ref[0])
    for n in ("idx", "w", "y", "g"):
        assert torch.equal(sv[n], ref[1][n]), n
    u = int(g["U"].item())
    assert u == int(ref[2]["U"].item())
    for n in ("dx", "dq", "dK1", "dK2", "dW1", "dW2", "dw"):
        assert torch.equal(g[n], ref[2][n]), n
    assert torch.equal(g["dV"][:u], ref[2]["dV"][:u]) and torch.equal(g["rows"][:u], ref[2]["rows"][:u])


@pytest.mark.parametrize("G,T_loc,B,N", [(2, 300, 32, 4096), (3, 257, 64, 1 << 20), (4, 64, 128, 512),
                                         (8, 77, 128, 1 << 26), (5, 1, 7, 3)])
def test_group_state_merge_bit_identical(G, T_loc, B, N):
    """The group's inverse map built once per group (each rank sorts its own
    positions, the sorted lists are merged: embbag_bwd_group_sort_local /
    _merge) equals one sort of all G*T_loc*B gathered positions
    (embbag_bwd_prepare): the bag backward from either state is
    bit-identical.  Skewed indices (many equal rows across ranks, so the merge's
    tie rule decides the order), G not a power of two, ragged tiles."""
    from paper_2412_09764_b200 import ops
    dv = 64
    rng = np.random.default_rng(G * 1000 + T_loc)
    hot = rng.integers(0, N, size=max(1, min(N, 50)))
    raw = np.where(rng.random((G * T_loc, B)) < 0.5, rng.choice(hot, size=(G * T_loc, B)),
                   rng.integers(0, N, size=(G * T_loc, B)))
    idx = torch.from_numpy(raw.astype(np.int32)).cuda()
    w = torch.from_numpy(rng.standard_normal((G * T_loc, B)).astype(np.float32)).cuda()
    dy = torch.from_numpy(rng.standard_normal((G * T_loc, dv)).astype(np.float32)).cuda().to(torch.bfloat16)
    V = torch.from_numpy(rng.standard_normal((N, dv)).astype(np.float32)).cuda().to(torch.bfloat16)
    ref_state = ops.embbag_bwd_prepare(N, dv, idx)
    lists = torch.empty((G, 2, T_loc * B), dtype=torch.int32, device="cuda")
    for g in range(G):
        ops.group_sort_local(N, idx[g * T_loc:(g + 1) * T_loc], g, out=lists[g])
    # each list: rows ascending, positions stable (ascending within a row) and global
    L = lists.cpu().numpy()
    for g in range(G):
        flat = raw[g * T_loc:(g + 1) * T_loc].reshape(-1)
        order = np.argsort(flat, kind="stable")
        assert np.array_equal(L[g, 0], flat[order]) and np.array_equal(L[g, 1], order + g * flat.size)
    state = ops.group_merge(N, dv, lists)
    a = ops.embbag_bwd(V, idx, w, dy, state=ref_state)
    b = ops.embbag_bwd(V, idx, w, dy, state=state)
    for x, y, n in zip(a, b, ("rows", "dV", "dw")):
        assert torch.equal(x, y), n


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_capi_group_p2p_equals_sendrecv(G):
    """The fused peer-memory exchanges (forward y blocks stored by the bag
    kernel into the owners' regions; backward dy slices stored by the pack
    kernel, partial dw blocks copied into the owners' slots and summed there
    in rank order) produce exactly the collective path's results (same
    arithmetic, same summation order), over three steps (both halves of every
    double-buffered section reused)."""
    from paper_2412_09764_b200 import ops
    T_loc, H, S, Dk, k, D = 64, 2, 64, 128, 8, 128
    # the full row and every rank's slice must pass the row-width rule
    # (bytes/16 a power of two or a multiple of 256)
    dv = 6144 if G == 3 else 128 * G
    h = _inputs(7, G * T_loc, H, S, Dk, dv, D)
    t = {n: torch.from_numpy(a).to(torch.bfloat16).cuda() for n, a in h.items()}
    hub = {p: ops.group_hub(G) for p in (False, True)}
    res = {False: [None] * G, True: [None] * G}
    errs = []

    def worker(r, p2p):
        try:
            torch.cuda.set_device(0)
            grp = ops.Group.from_hub(hub[p2p], r).set_p2p(p2p)
            with torch.cuda.stream(torch.cuda.Stream()):
                sl = slice(r * T_loc, (r + 1) * T_loc)
                lo, hi = r * dv // G, (r + 1) * dv // G
                Vs = t["V"][:, lo:hi].contiguous()
                x, q, dout = (t[n][sl].contiguous() for n in ("x", "q", "dout"))
                outs = []
                for step in range(3):
                    xs = x * (1 + step)        # a different forward every step
                    out, sv = ops.memory_layer_fwd_group(grp, xs, q, t["K1"], t["K2"], Vs, t["W1"],
                                                         t["W2"], k, mode="alltoall")
                    g = ops.memory_layer_bwd_group(grp, dout, xs, q, t["K1"], t["K2"], Vs, t["W1"],
                                                   t["W2"], sv, want_dw=True)
                    torch.cuda.current_stream().synchronize()
                    outs.append((out.clone(), sv["y"].clone(), g["dw"].clone(), g["dq"].clone(),
                                 g["dx"].clone()))
                res[p2p][r] = outs
            grp.close()
        except Exception as e:  # surface thread failures
            errs.append(e)

    for p2p in (False, True):
        ths = [threading.Thread(target=worker, args=(r, p2p)) for r in range(G)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        ops.group_hub_destroy(hub[p2p])
    assert not errs, errs
    for r in range(G):
        for a, b in zip(res[False][r], res[True][r]):
            for x, y in zip(a, b):
                assert torch.equal(x, y)


def test_loopback_group_uses_captures():
    """ml_group_init_loopback (t_ref(G) through the library's group path):
    rank 0 of a G = 2 group on one GPU, the other rank's (idx, w) and sorted
    lists taken from a hub run's captures -- the gathered indices, the
    inverse map (distinct rows U, the rows) and rank 0's own outputs that do
    not depend on the other rank's data (idx, w of its own tokens) match the
    hub run exactly."""
    from paper_2412_09764_b200 import ops
    G, T_loc, H, S, Dk, k, D = 2, 64, 2, 64, 128, 8, 128
    dv = 256
    h = _inputs(9, G * T_loc, H, S, Dk, dv, D)
    t = {n: torch.from_numpy(a).to(torch.bfloat16).cuda() for n, a in h.items()}
    res = _run_hub(t, G, T_loc, dv, k, "alltoall")
    out0, sv0, g0 = res[0]
    B = H * k
    idx_all, w_all = sv0["idx_all"], sv0["w_all"]
    lists = torch.empty((G, 2, T_loc * B), dtype=torch.int32, device="cuda")
    for r in range(G):
        ops.group_sort_local(S * S, idx_all[r * T_loc:(r + 1) * T_loc].reshape(T_loc, B), r, out=lists[r])
    n = idx_all.shape[0]
    iw = torch.cat([idx_all.reshape(n, -1), w_all.reshape(n, -1).view(torch.int32)], 1).contiguous()
    grp = ops.Group.loopback(G, 0, [iw, lists])
    sl = slice(0, T_loc)
    Vs = t["V"][:, :dv // G].contiguous()
    x, q, dout = (t[nm][sl].contiguous() for nm in ("x", "q", "dout"))
    out, sv = ops.memory_layer_fwd_group(grp, x, q, t["K1"], t["K2"], Vs, t["W1"], t["W2"], k)
    g = ops.memory_layer_bwd_group(grp, dout, x, q, t["K1"], t["K2"], Vs, t["W1"], t["W2"], sv,
                                   want_dw=True)
    torch.cuda.synchronize()
    assert torch.equal(sv["idx"], sv0["idx"]) and torch.equal(sv["w"], sv0["w"])
    assert torch.equal(sv["idx_all"], idx_all) and torch.equal(sv["w_all"], w_all)
    u, u0 = int(g["U"].item()), int(g0["U"].item())
    assert u == u0 and torch.equal(g["rows"][:u], g0["rows"][:u0])
    assert torch.isfinite(out.float()).all() and torch.isfinite(g["dq"]).all()
    grp.close()
