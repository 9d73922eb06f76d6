"""The dim-sharded memory-group protocol (Fig. 2) under
torch.distributed gloo, world size 2, on CPU: two processes run
paper_2412_09764_b200.group.GroupMemoryLayer with the oracle as the local
compute, and the result must equal the unsharded memory layer (oracle):
own-token outputs and gradients, dV shards = column slices of dV, dK summed
over ranks = dK."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import layer as olayer
from synthetic import gen

T_LOC, H, S, DK, K, DV, D = 6, 2, 8, 8, 3, 8, 6


def _inputs(G):
    f = lambda tag, shape: gen.tensor(5, tag, shape).astype(np.float64)
    T = G * T_LOC
    return dict(x=f("x", (T, D)), q=f("q", (T, H, DK)), K1=f("K1", (H, S, DK // 2)),
                K2=f("K2", (H, S, DK // 2)), V=f("V", (S * S, DV)), W1=f("W1", (D, DV)),
                W2=f("W2", (DV, D)), dout=f("dout", (T, D)))


def _worker(rank, G, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=G)
    try:
        from paper_2412_09764_b200.group import GroupMemoryLayer
        from tests.group_oracle_local import OracleLocal
        p = _inputs(G)
        sl = slice(rank * T_LOC, (rank + 1) * T_LOC)
        lo, hi = rank * DV // G, (rank + 1) * DV // G
        t = {n: torch.from_numpy(np.ascontiguousarray(a)) for n, a in p.items()}
        layer = GroupMemoryLayer(None, K, mode=mode, local=OracleLocal())
        out, saved = layer.forward(t["x"][sl], t["q"][sl], t["K1"], t["K2"],
                                   t["V"][:, lo:hi].contiguous(), t["W1"], t["W2"])
        g = layer.backward(t["dout"][sl].contiguous(), saved)
        res = dict(out=out.numpy(), dq=g["dq"].numpy(), dx=g["dx"].numpy(), dK1=g["dK1"].numpy(),
                   dK2=g["dK2"].numpy(), dW1=g["dW1"].numpy(), dW2=g["dW2"].numpy(),
                   rows=g["rows"].numpy(), dV=g["dV"].numpy(), dw=g["dw"].numpy(),
                   y_all=None if saved["y_all"] is None else saved["y_all"].numpy())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("mode", ["alltoall", "allgather"])
def test_group_protocol_gloo_world2(mode):
    G = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, G, port, mode, q)) for r in range(G)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(G))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = _inputs(G)
    out, saved = olayer.memory_layer_fwd(p["x"], p["q"], p["K1"], p["K2"], p["V"], p["W1"], p["W2"], K)
    ref = olayer.memory_layer_bwd(p["dout"], p["x"], p["q"], p["K1"], p["K2"], p["V"], p["W1"],
                                  p["W2"], saved)
    tol = dict(rtol=1e-10, atol=1e-12)
    for r in range(G):
        sl = slice(r * T_LOC, (r + 1) * T_LOC)
        lo, hi = r * DV // G, (r + 1) * DV // G
        np.testing.assert_allclose(res[r]["out"], out[sl], **tol)
        np.testing.assert_allclose(res[r]["dq"], ref["dq"][sl], **tol)
        np.testing.assert_allclose(res[r]["dx"], ref["dx"][sl], **tol)
        np.testing.assert_allclose(res[r]["dw"], ref["dw"][sl], **tol)
        assert np.array_equal(res[r]["rows"], ref["rows"])          # every shard sees all rows
        np.testing.assert_allclose(res[r]["dV"], ref["dV"][:, lo:hi], **tol)
        if mode == "allgather":
            np.testing.assert_allclose(res[r]["y_all"], saved["y"], **tol)
    np.testing.assert_allclose(res[0]["dK1"] + res[1]["dK1"], ref["dK1"], **tol)
    np.testing.assert_allclose(res[0]["dK2"] + res[1]["dK2"], ref["dK2"], **tol)
    np.testing.assert_allclose(res[0]["dW1"] + res[1]["dW1"], ref["dW1"], **tol)
    np.testing.assert_allclose(res[0]["dW2"] + res[1]["dW2"], ref["dW2"], **tol)
