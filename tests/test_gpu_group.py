"""Memory group on one GPU: G simulated ranks as host threads (each with its
own CUDA stream) exchanging through an in-process communicator, running the
real CUDA local ops (pack/unpack kernels, sharded bag fwd/bwd, pkm).  Kernels
never wait on each other on the device (the exchange is host-synchronised).
Checks sharded == unsharded: y and dV bit-exact (each element
keeps its accumulation order under column sharding), out / dw / dq / dK /
dW within tolerance (re-associated sums and different GEMM shapes)."""
import threading

import numpy as np
import pytest
import torch

from oracle import group as ogroup, layer as olayer
from synthetic import gen
from tests.gpu_util import TOL, assert_close, compare_topk, host, layer_magnitudes

pytestmark = pytest.mark.gpu


class ThreadComm:
    def __init__(self, G, rank, shared):
        self.size, self.rank, self.sh = G, rank, shared

    def _publish(self, t):
        torch.cuda.current_stream().synchronize()
        self.sh["slots"][self.rank] = t
        self.sh["bar"].wait()

    def _done(self):
        torch.cuda.current_stream().synchronize()
        self.sh["bar"].wait()

    def all_gather(self, out, inp):
        self._publish(inp.contiguous())
        out.copy_(torch.cat([s for s in self.sh["slots"]], 0).view(out.shape))
        self._done()

    def all_to_all(self, out, inp):
        self._publish(inp.contiguous())
        n = inp.shape[0] // self.size
        out.copy_(torch.cat([s[self.rank * n:(self.rank + 1) * n] for s in self.sh["slots"]], 0))
        self._done()

    def reduce_scatter(self, out, inp):
        self._publish(inp.contiguous())
        n = out.shape[0]
        acc = self.sh["slots"][0][self.rank * n:(self.rank + 1) * n].clone()
        for s in self.sh["slots"][1:]:
            acc += s[self.rank * n:(self.rank + 1) * n]
        out.copy_(acc)
        self._done()


def _inputs(seed, T, H, S, Dk, dv, D, dt="bf16"):
    f = lambda tag, shape, sc=1.0: gen.tensor(seed, tag, shape, scale=sc, dtype=dt)
    return dict(x=f("x", (T, D)), q=f("q", (T, H, Dk)),
                K1=f("K1", (H, S, Dk // 2), gen.scale_for("K1", Dk=Dk)),
                K2=f("K2", (H, S, Dk // 2), gen.scale_for("K2", Dk=Dk)),
                V=f("V", (S * S, dv)), W1=f("W1", (D, dv), gen.scale_for("W1", D=D)),
                W2=f("W2", (dv, D), gen.scale_for("W2", dv=dv)), dout=f("dout", (T, D)))


@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("mode", ["alltoall", "allgather"])
def test_group_sharded_equals_unsharded(G, mode):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_09764_b200 import ops
    from paper_2412_09764_b200.group import GroupMemoryLayer
    T_loc, H, S, Dk, k, dv, D = 96, 4, 64, 128, 8, 512, 256
    T = G * T_loc
    h = _inputs(3, T, H, S, Dk, dv, D)
    t = {n: torch.from_numpy(a).to(torch.bfloat16).cuda() for n, a in h.items()}
    out, saved = ops.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"], k)
    ref = ops.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                               t["W2"], saved, want_dw=True)
    U = int(ref["U"].item())
    torch.cuda.synchronize()
    shared = {"slots": [None] * G, "bar": threading.Barrier(G)}
    res, errs = [None] * G, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                sl = slice(r * T_loc, (r + 1) * T_loc)
                lo, hi = r * dv // G, (r + 1) * dv // G
                layer = GroupMemoryLayer(ThreadComm(G, r, shared), k, mode=mode)
                Vs = t["V"][:, lo:hi].contiguous()
                o, sv = layer.forward(t["x"][sl].contiguous(), t["q"][sl].contiguous(), t["K1"],
                                      t["K2"], Vs, t["W1"], t["W2"])
                g = layer.backward(t["dout"][sl].contiguous(), sv)
                torch.cuda.current_stream().synchronize()
                res[r] = (o, sv, g)
        except Exception as e:  # surface thread failures
            errs.append(e)
            shared["bar"].abort()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errs, errs
    dK1 = sum(host(res[r][2]["dK1"]) for r in range(G))
    dK2 = sum(host(res[r][2]["dK2"]) for r in range(G))
    dW1 = sum(host(res[r][2]["dW1"]) for r in range(G))
    dW2 = sum(host(res[r][2]["dW2"]) for r in range(G))
    for r in range(G):
        o, sv, g = res[r]
        sl = slice(r * T_loc, (r + 1) * T_loc)
        lo, hi = r * dv // G, (r + 1) * dv // G
        assert torch.equal(sv["idx"], saved["idx"][sl])
        assert torch.equal(sv["y"], saved["y"][sl])                    # bit-exact
        if mode == "allgather":
            assert torch.equal(sv["y_all"], saved["y"])
        u = int(g["U"].item())
        assert u == U and torch.equal(g["rows"][:u], ref["rows"][:U])
        assert torch.equal(g["dV"][:u], ref["dV"][:U, lo:hi])          # bit-exact
    # out / dw / dq / dx / dK / dW: re-associated sums and different GEMM
    # shapes (a bf16 rounding of dz / dy can flip) -> checked against the
    # oracle below with the rounding-model bound

    # every rank against the fp64 oracle: the group protocol (oracle/group.py,
    # P:167) for the bag output of each rank, the plain layer (oracle/layer.py)
    # for the rest (sharded == unsharded, S:411 / S:429)
    h64 = {n: a.astype(np.float64) for n, a in h.items()}
    rout, rs = olayer.memory_layer_fwd(h64["x"], h64["q"], h64["K1"], h64["K2"], h64["V"],
                                       h64["W1"], h64["W2"], k)
    assert not compare_topk(host(saved["idx"]), rs["idx"], h64["q"], h64["K1"], h64["K2"])
    rb = olayer.memory_layer_bwd(h64["dout"], h64["x"], h64["q"], h64["K1"], h64["K2"], h64["V"],
                                 h64["W1"], h64["W2"], rs)
    m = layer_magnitudes(h64, rs, rb)
    B = H * k
    idx_r = [rs["idx"][r * T_loc:(r + 1) * T_loc].reshape(T_loc, B) for r in range(G)]
    w_r = [rs["w"][r * T_loc:(r + 1) * T_loc].reshape(T_loc, B) for r in range(G)]
    ry = ogroup.group_fwd(h64["V"], idx_r, w_r, G, mode=mode)
    for r in range(G):
        o, sv, g = res[r]
        sl = slice(r * T_loc, (r + 1) * T_loc)
        lo, hi = r * dv // G, (r + 1) * dv // G
        want_y = ry[r] if mode == "alltoall" else ry[r][sl]
        my = m["y"] if mode == "allgather" else m["y"][sl]
        assert_close(host(sv["y"]), want_y, TOL["bf16"], f"y rank {r}", mag=m["y"][sl])
        if mode == "allgather":
            assert_close(host(sv["y_all"]), ry[r], TOL["bf16"], f"y_all rank {r}", mag=my)
        assert_close(host(o), rout[sl], TOL["bf16"], f"out rank {r}", mag=m["out"][sl])
        u = int(g["U"].item())
        assert np.array_equal(host(g["rows"][:u]), rb["rows"])
        assert_close(host(g["dV"][:u]), rb["dV"][:, lo:hi], TOL["bf16"], f"dV shard {r}",
                     mag=m["dV"][:, lo:hi])
        for n in ("dw", "dq", "dx"):
            assert_close(host(g[n]), rb[n][sl], TOL["bf16"], f"{n} rank {r}", mag=m[n][sl])
    for n, got in (("dK1", dK1), ("dK2", dK2), ("dW1", dW1), ("dW2", dW2)):
        assert_close(got, rb[n], TOL["bf16"], f"{n} vs oracle", mag=m[n])
