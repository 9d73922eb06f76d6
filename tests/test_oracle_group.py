"""Pins of oracle/group.py: the sharded protocol of P:167 / Fig. 2 equals the
unsharded bag, bit-exact on the dyadic class for
G in {1,2,4,8}; dw equal to rounding on continuous inputs."""
import numpy as np
import pytest

from oracle import bag, group
from synthetic import gen, streams


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", ["alltoall", "allgather"])
def test_sharded_equals_unsharded(G, mode):
    N, dv, T_loc, B = 128, 16, 5, 6
    V = gen.tensor(G, "V", (N, dv), cls=gen.CLS_EXACT).astype(np.float64)
    idx = [streams.uniform_indices(100 + r, T_loc, B, N) for r in range(G)]
    w = [streams.softmax_free_weights(100 + r, T_loc, B, cls=gen.CLS_DYADIC).astype(np.float64)
         for r in range(G)]
    outs = group.group_fwd(V, idx, w, G, mode)
    y_all = bag.embbag_fwd(V, np.concatenate(idx), np.concatenate(w))
    for r in range(G):
        want = y_all if mode == "allgather" else y_all[r * T_loc:(r + 1) * T_loc]
        assert np.array_equal(outs[r], want)
    dy_all = gen.tensor(G, "dout", (G * T_loc, dv), cls=gen.CLS_EXACT).astype(np.float64)
    dy = [dy_all] * G if mode == "allgather" else [dy_all[r * T_loc:(r + 1) * T_loc] for r in range(G)]
    shards, dw = group.group_bwd(V, idx, w, dy, G, mode)
    rows, dV, dw_ref = bag.embbag_bwd(V, np.concatenate(idx), np.concatenate(w), dy_all)
    for g, (lo, hi) in enumerate(group.shard_columns(dv, G)):
        assert np.array_equal(shards[g][0], rows)
        assert np.array_equal(shards[g][1], dV[:, lo:hi])
    np.testing.assert_array_equal(np.concatenate(dw), dw_ref)


def test_bad_group_size():
    with pytest.raises(ValueError):
        group.shard_columns(10, 4)
