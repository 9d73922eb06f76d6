"""Parallel memory: the value table sharded along the embedding dim over a
memory group (§3.1.2; Fig. 2 caption P:162).

"The memory values are sharded across the embedding dimension.  At each
step, the indices are gathered from the process group, each worker does a
lookup and then aggregates the portion of embeddings in its own shard.  After
this, each worker gathers the partial embeddings corresponding to its own
portion of the indices."

Forward per rank (T_loc own tokens, shard V_g = V[:, g*dv/G:(g+1)*dv/G]):
  1. idx, w = pkm_topk(own queries)                         (own tokens only)
  2. all-gather (idx, w) over the group                     [G*T_loc, H*k]
  3. y_part = embbag over V_g for ALL group tokens          [G*T_loc, dv/G]
  4. mode "alltoall" (paper): all-to-all so each rank gets the G slices of
     its own tokens, unpacked into [T_loc, dv] with the silu gate fused;
     mode "allgather" (north-star wording): all-gather of every slice, every
     rank unpacks all tokens [G*T_loc, dv]
  5. out = (y * silu(x W1)) W2 on own tokens
Backward (reverse, reading Q14 in DESIGN.md): gate backward on own tokens,
all-to-all of the dy slices, local sorted backward on V_g (dV never leaves
the rank), reduce-scatter of the partial dw (a dot over dv/G columns) to the
token owners, then the key/query backward on own tokens.

The exchange goes through a `comm` object (torch.distributed: NCCL on GPUs,
gloo in the CPU tests); the local compute goes through `local` (the CUDA
kernels of libmemlayer via ops.py).  Both are injectable so the protocol is
tested on CPU with world size 2 (tests/test_group_gloo.py).
"""
import torch


class TorchComm:
    """Collectives of one process group (torch.distributed)."""

    def __init__(self, pg=None):
        import torch.distributed as dist
        self.dist = dist
        self.pg = pg
        self.size = dist.get_world_size(pg)
        self.rank = dist.get_rank(pg)

    def all_gather(self, out, inp):
        """out [G*n, ...] <- concatenation of every rank's inp [n, ...]."""
        self.dist.all_gather_into_tensor(out, inp.contiguous(), group=self.pg)

    def all_to_all(self, out, inp):
        """Chunk g (dim 0, equal split) of inp goes to rank g; out chunk g
        comes from rank g."""
        self.dist.all_to_all_single(out, inp.contiguous(), group=self.pg)

    def reduce_scatter(self, out, inp):
        """out [n, ...] = sum over ranks of chunk `rank` of inp [G*n, ...]."""
        self.dist.reduce_scatter_tensor(out, inp.contiguous(), group=self.pg)


class CudaLocal:
    """Local compute on this rank's GPU through the C ABI (ops.py)."""

    grad_dtype = torch.float32

    def __init__(self, dV_dtype=torch.float32):
        from . import ops
        self.ops = ops
        self._side = None
        self.dV_dtype = dV_dtype        # storage of the compact value gradient (memlayer.h)

    def empty(self, shape, dtype, like):
        return torch.empty(shape, dtype=dtype, device=like.device)

    # ---- side stream: work that only depends on already computed tensors
    # (the inverse index map during the forward, the gate weight gradients
    # during the exchange + bag backward) runs concurrently on a
    # high-priority stream; join() makes the current stream wait for it.
    def side(self, like):
        cur = torch.cuda.current_stream(like.device)
        if self.ops.SERIAL:       # measurement mode: one in-order stream
            return torch.cuda.stream(cur)
        if self._side is None:
            self._side = torch.cuda.Stream(device=like.device, priority=-100)   # the highest
        self._side.wait_stream(cur)
        return torch.cuda.stream(self._side)

    def join(self, *tensors):
        if self._side is None:
            return
        cur = torch.cuda.current_stream()
        cur.wait_stream(self._side)
        for t in tensors:
            if t is not None:
                t.record_stream(cur)

    def embbag_bwd_prepare(self, N, dv, idx, dtype):
        """The backward's inverse map on a normal-priority background stream
        (it fills SMs the forward's tail leaves idle); returns (state, event):
        the backward waits on the event, the forward does not."""
        cur = torch.cuda.current_stream(idx.device)
        if self.ops.SERIAL:       # measurement mode: one in-order stream
            state = self.ops.embbag_bwd_prepare(N, dv, idx, dtype)
            ev = torch.cuda.Event()
            ev.record(cur)
            return state, ev
        if getattr(self, "_bg", None) is None:
            self._bg = torch.cuda.Stream(device=idx.device)
        self._bg.wait_stream(cur)           # also orders it after the previous backward
        with torch.cuda.stream(self._bg):
            # one persistent state buffer (allocated once, on this stream)
            state = self.ops.embbag_bwd_prepare(N, dv, idx, dtype, out=getattr(self, "_state", None))
            self._state = state
            ev = torch.cuda.Event()
            ev.record(self._bg)
        idx.record_stream(self._bg)
        return state, ev

    # ---- the group's inverse map, built once per group (include/memlayer.h
    # embbag_bwd_group_sort_local / _merge): own positions sorted on the
    # background stream during the forward, the G sorted lists exchanged at
    # the end of the forward, merged on the background stream
    def _bg_stream(self, like):
        cur = torch.cuda.current_stream(like.device)
        if self.ops.SERIAL:       # measurement mode: one in-order stream
            return cur
        if getattr(self, "_bg", None) is None:
            self._bg = torch.cuda.Stream(device=like.device)
        self._bg.wait_stream(cur)
        return self._bg

    def group_sort_local(self, N, idx, rank):
        bg = self._bg_stream(idx)
        with torch.cuda.stream(bg):
            lst = getattr(self, "_lst", None)
            if lst is None or lst.shape[1] != idx.numel():
                lst = self._lst = torch.empty((2, idx.numel()), dtype=torch.int32, device=idx.device)
                self._lst_ws = None
            self.ops.group_sort_local(N, idx, rank, out=lst, ws=getattr(self, "_lst_ws", None))
            self._sorted_ev = torch.cuda.Event()
            self._sorted_ev.record(bg)
        if bg is not torch.cuda.current_stream(idx.device):
            idx.record_stream(bg)
        return lst

    def group_lists(self, G, lst):
        buf = getattr(self, "_lists", None)
        if buf is None or buf.shape != (G,) + tuple(lst.shape):
            buf = self._lists = torch.empty((G,) + tuple(lst.shape), dtype=lst.dtype, device=lst.device)
        torch.cuda.current_stream(lst.device).wait_event(self._sorted_ev)
        return buf

    def group_merge(self, N, dv, lists, dtype):
        bg = self._bg_stream(lists)
        with torch.cuda.stream(bg):
            state = self.ops.group_merge(N, dv, lists, dtype, out=getattr(self, "_state", None))
            self._state = state
            ev = torch.cuda.Event()
            ev.record(bg)
        return state, ev

    def wait(self, ev):
        torch.cuda.current_stream().wait_event(ev)

    def pkm_topk(self, q, K1, K2, k):
        return self.ops.pkm_topk(q, K1, K2, k)

    def embbag_fwd(self, V, idx, w):
        return self.ops.embbag_fwd(V, idx, w)

    def embbag_bwd(self, V, idx, w, dy, state=None):
        # outputs reused across calls (valid until the next backward): the
        # capacity-sized dV is the largest allocation of the step
        if not hasattr(self, "_bufs"):
            self._bufs = {}
        rows, dV, U, dw = self.ops.embbag_bwd(V, idx, w, dy, sync=False, state=state,
                                              grad_dtype=self.dV_dtype, bufs=self._bufs)
        return rows, dV, U, dw

    def pkm_topk_bwd(self, q, K1, K2, idx, w, dw, dK1, dK2):
        return self.ops.pkm_topk_bwd(q, K1, K2, idx, w, dw, dK1, dK2)

    def gemm(self, A, B, transA=False, transB=False, out_f32=False):
        return self.ops.gemm(A, B, transA, transB, out_f32)

    def unpack(self, recv, G, T_loc, dv, gate=None, want_y=True):
        return self.ops.group_unpack(recv, G, T_loc, dv, gate, want_y)

    def pack(self, src, G):
        return self.ops.group_pack(src, G)

    def gate_bwd(self, dz, g, y):
        return self.ops.gate_bwd(dz, g, y)


def shard_bounds(dv, G, rank):
    if dv % G:
        raise ValueError("G must divide the value dim (SPEC S:401)")
    w = dv // G
    return rank * w, (rank + 1) * w


class GroupMemoryLayer:
    """Memory+ layer whose value table is dim-sharded over a memory group."""

    def __init__(self, comm, k, mode="alltoall", local=None):
        if mode not in ("alltoall", "allgather"):
            raise ValueError(mode)
        self.comm = comm if hasattr(comm, "all_to_all") else TorchComm(comm)
        self.k = k
        self.mode = mode
        self.local = local or CudaLocal()

    def forward(self, x, q, K1, K2, V_shard, W1, W2):
        L, C, k = self.local, self.comm, self.k
        G, rank = C.size, C.rank
        T_loc, H, _ = q.shape
        B = H * k
        dvG = V_shard.shape[1]
        dv = dvG * G
        idx, w = L.pkm_topk(q, K1, K2, k)                              # 1
        # the backward's inverse map, built once per group: own positions
        # sorted now (beside the exchange and the bag forward), the G sorted
        # lists exchanged and merged at the end of the forward
        lst = L.group_sort_local(V_shard.shape[0], idx.view(T_loc, B), rank) \
            if hasattr(L, "group_sort_local") else None
        idx_all = L.empty((G * T_loc, H, k), idx.dtype, idx)
        w_all = L.empty((G * T_loc, H, k), w.dtype, w)
        C.all_gather(idx_all, idx)                                      # 2
        C.all_gather(w_all, w)
        y_part = L.embbag_fwd(V_shard, idx_all.view(G * T_loc, B), w_all.view(G * T_loc, B))  # 3
        gpre = L.gemm(x, W1)
        if self.mode == "alltoall":                                     # 4 (paper)
            recv = L.empty(y_part.shape, y_part.dtype, y_part)
            C.all_to_all(recv, y_part)
            y, z = L.unpack(recv.view(G, T_loc, dvG), G, T_loc, dv, gate=gpre)
            y_all = None
        else:                                                           # 4 (north star)
            full = L.empty((G * G * T_loc, dvG), y_part.dtype, y_part)
            C.all_gather(full, y_part)
            y_all, _ = L.unpack(full.view(G, G * T_loc, dvG), G, G * T_loc, dv)
            y = y_all[rank * T_loc:(rank + 1) * T_loc]
            _, z = L.unpack(y.reshape(1, T_loc, dv), 1, T_loc, dv, gate=gpre, want_y=False)
        out = L.gemm(z, W2)                                             # 5
        state = state_ev = None
        if lst is not None:
            lists = L.group_lists(G, lst)
            C.all_gather(lists, lst.unsqueeze(0))                      # [G, 2, T_loc*B]
            state, state_ev = L.group_merge(V_shard.shape[0], dvG, lists, V_shard.dtype)
        saved = dict(x=x, q=q, K1=K1, K2=K2, V=V_shard, W1=W1, W2=W2, idx=idx, w=w,
                     idx_all=idx_all, w_all=w_all, g=gpre, y=y, y_all=y_all, state=state,
                     state_ev=state_ev)
        return out, saved

    def backward(self, dout, saved, dK1=None, dK2=None):
        L, C, k = self.local, self.comm, self.k
        G = C.size
        q, V_shard = saved["q"], saved["V"]
        T_loc, H, _ = q.shape
        B = H * k
        dvG = V_shard.shape[1]
        dz = L.gemm(dout, saved["W2"], transB=True)                     # gate backward
        z, dy, dg = L.gate_bwd(dz, saved["g"], saved["y"])
        side = hasattr(L, "side")
        if side:      # gate weight gradients overlap the exchange and the bag backward
            with L.side(dz):
                dW2 = L.gemm(z, dout, transA=True, out_f32=True)
                dW1 = L.gemm(saved["x"], dg, transA=True, out_f32=True)
                dx = L.gemm(dg, saved["W1"], transB=True)
        else:
            dW2 = L.gemm(z, dout, transA=True, out_f32=True)
            dW1 = L.gemm(saved["x"], dg, transA=True, out_f32=True)
            dx = L.gemm(dg, saved["W1"], transB=True)
        send = L.pack(dy, G)                                            # [G, T_loc, dv/G]
        recv = L.empty((G * T_loc, dvG), dy.dtype, dy)
        C.all_to_all(recv, send.view(G * T_loc, dvG))                  # dy slices of all tokens
        bag_args = (V_shard, saved["idx_all"].view(G * T_loc, B), saved["w_all"].view(G * T_loc, B),
                    recv)
        if saved.get("state") is not None:
            L.wait(saved["state_ev"])              # the forward's state build is complete
            rows, dV, U, dw_part = L.embbag_bwd(*bag_args, state=saved["state"])
        else:
            rows, dV, U, dw_part = L.embbag_bwd(*bag_args)
        dw = L.empty((T_loc, B), dw_part.dtype, dw_part)
        C.reduce_scatter(dw, dw_part)                                   # sum over column shards
        if dK1 is None:
            dK1 = torch.zeros(saved["K1"].shape, dtype=L.grad_dtype, device=dw.device)
        if dK2 is None:
            dK2 = torch.zeros(saved["K2"].shape, dtype=L.grad_dtype, device=dw.device)
        dq, dK1, dK2 = L.pkm_topk_bwd(q, saved["K1"], saved["K2"], saved["idx"], saved["w"],
                                      dw.view(T_loc, H, k), dK1, dK2)
        if side:
            L.join(dW1, dW2, dx, z, dg)
        return dict(dx=dx, dq=dq, dK1=dK1, dK2=dK2, dW1=dW1, dW2=dW2, rows=rows, dV=dV, U=U,
                    dw=dw.view(T_loc, H, k))


# --------------------------------------------------------------- C-ABI group
def nccl_group(pg=None):
    """Bootstraps the library's NCCL memory group (include/memlayer.h
    ml_group_init) over a torch.distributed process group: rank 0 creates the
    128-byte ncclUniqueId, torch.distributed broadcasts it."""
    import torch.distributed as dist
    from . import ops
    rank, G = dist.get_rank(pg), dist.get_world_size(pg)
    obj = [ops.group_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(pg, 0) if pg is not None else 0, group=pg)
    return ops.Group.nccl(obj[0], G, rank)


class CGroupMemoryLayer:
    """The memory group through the C ABI (memory_layer_fwd_group /
    memory_layer_bwd_group): the exchange, its overlap with the bag forward
    and all local kernels run inside the library."""

    def __init__(self, grp, k, mode="alltoall", dV_dtype=torch.float32):
        if mode not in ("alltoall", "allgather"):
            raise ValueError(mode)
        self.grp, self.k, self.mode, self.dV_dtype = grp, k, mode, dV_dtype
        self.bufs = {}      # backward outputs, reused across steps (valid until the next one)
        self.fbufs = {}     # forward outputs / saved tensors, likewise

    def forward(self, x, q, K1, K2, V_shard, W1, W2):
        from . import ops
        out, saved = ops.memory_layer_fwd_group(self.grp, x, q, K1, K2, V_shard, W1, W2, self.k,
                                                mode=self.mode, bufs=self.fbufs)
        saved.update(x=x, q=q, K1=K1, K2=K2, V=V_shard, W1=W1, W2=W2)
        return out, saved

    def backward(self, dout, saved, dK1=None, dK2=None):
        from . import ops
        return ops.memory_layer_bwd_group(self.grp, dout, saved["x"], saved["q"], saved["K1"],
                                          saved["K2"], saved["V"], saved["W1"], saved["W2"], saved,
                                          dK1=dK1, dK2=dK2, dV_dtype=self.dV_dtype, want_dw=True,
                                          bufs=self.bufs)
