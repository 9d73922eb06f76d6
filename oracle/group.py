"""Parallel memory, §3.1.2 (Fig. 2 caption P:162),
simulated sequentially for G ranks.

"The memory values are sharded across the embedding dimension.  At each
step, the indices are gathered from the process group, each worker does a
lookup and then aggregates the portion of embeddings in its own shard.  After
this, each worker gathers the partial embeddings corresponding to its own
portion of the indices."

Two output modes (reading Q13): "alltoall" (the paper: each rank receives
only its own tokens' full rows) and "allgather" (the north-star wording:
every rank receives all tokens' full rows).  Backward (reading Q14): the
reverse exchange; dV never leaves its shard; dw partials (dots over a column
slice) are summed over shards.
"""
import numpy as np

from . import bag


def shard_columns(dv, G):
    if dv % G:
        raise ValueError("G must divide the value dim (S:401)")
    w = dv // G
    return [(g * w, (g + 1) * w) for g in range(G)]


def _slice_V(V, lo, hi):
    if callable(V):
        return lambda ids: np.asarray(V(ids))[:, lo:hi]
    return np.asarray(V)[:, lo:hi]


def group_fwd(V, idx_per_rank, w_per_rank, G, mode="alltoall"):
    """Returns the per-rank outputs: alltoall -> [T_loc, dv] of the rank's own
    tokens; allgather -> [G*T_loc, dv] of all tokens."""
    cols = shard_columns(_dv(V, idx_per_rank), G)
    idx_all = np.concatenate(idx_per_rank, axis=0)   # phase 1: all-gather
    w_all = np.concatenate(w_per_rank, axis=0)
    T_loc = idx_per_rank[0].shape[0]
    partial = [bag.embbag_fwd(_slice_V(V, lo, hi), idx_all, w_all)   # phase 2
               for (lo, hi) in cols]
    full = np.concatenate(partial, axis=1)
    if mode == "allgather":
        return [full.copy() for _ in range(G)]
    return [full[r * T_loc:(r + 1) * T_loc] for r in range(G)]      # phase 3


def group_bwd(V, idx_per_rank, w_per_rank, dy_per_rank, G, mode="alltoall"):
    """Per-shard (rows, dV_slice) and per-rank dw (summed over shards).
    dy_per_rank: alltoall -> each rank's own tokens [T_loc, dv];
    allgather -> every rank holds dy for all tokens (identical copies)."""
    dv = _dv(V, idx_per_rank)
    cols = shard_columns(dv, G)
    idx_all = np.concatenate(idx_per_rank, axis=0)
    w_all = np.concatenate(w_per_rank, axis=0)
    T_loc = idx_per_rank[0].shape[0]
    if mode == "allgather":
        dy_all = np.asarray(dy_per_rank[0], np.float64)
    else:
        dy_all = np.concatenate(dy_per_rank, axis=0)
    shards = []
    dw_sum = np.zeros(idx_all.shape)
    for (lo, hi) in cols:
        rows, dV, dw_part = bag.embbag_bwd(_slice_V(V, lo, hi), idx_all, w_all,
                                           dy_all[:, lo:hi])
        shards.append((rows, dV))
        dw_sum += dw_part
    dw = [dw_sum[r * T_loc:(r + 1) * T_loc] for r in range(G)]
    return shards, dw


def _dv(V, idx_per_rank):
    if callable(V):
        return np.asarray(V(np.asarray([idx_per_rank[0].reshape(-1)[0]]))).shape[1]
    return np.asarray(V).shape[1]
