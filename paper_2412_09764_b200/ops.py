"""Torch-facing binding of libmemlayer: argument marshalling only.

Every function checks dtype/device/contiguity, allocates outputs with torch
(device memory is PyTorch's job here), and calls the C ABI on the current
CUDA stream.  No arithmetic of the method happens in Python.  Names follow
include/memlayer.h.
"""
import ctypes as C
import weakref

import torch

from . import _lib
from ._lib import PkmShape, BagShape, LayerShape, PeerShape, check, lib

_DT = {torch.bfloat16: _lib.ML_BF16, torch.float32: _lib.ML_F32}
_WS = {}
SERIAL = False      # set_serial(): measurement mode, no side-stream concurrency


def _dt(t):
    if t.dtype not in _DT:
        raise TypeError(f"unsupported dtype {t.dtype} (bf16 or fp32)")
    return _DT[t.dtype]


def _p(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("tensor must be on a CUDA device")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def workspace(nbytes, device=None, tag="default"):
    """A cached uint8 device buffer of at least nbytes (grown on demand), one
    per (device, tag, current stream) so concurrent streams never share it."""
    device = torch.device(device or torch.cuda.current_device())
    key = (device.index, tag, torch.cuda.current_stream(device).cuda_stream)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        _WS.pop(key, None)
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def release_workspaces():
    """Drop the cached workspaces.  Must not be called while a captured
    MemoryLayerStepGraph (graph.py) is alive: the graph replays kernels whose
    workspace pointers were baked in at capture time."""
    _WS.clear()


def launch_count():
    """Kernels launched by libmemlayer since it was loaded."""
    return int(lib().ml_launch_count())


def timing_enable(on=True):
    lib().ml_timing_enable(1 if on else 0)


def set_serial(on=True):
    """Measurement only: issue every kernel of a layer call on the caller's
    stream (no auxiliary-stream concurrency) so per-launch timing events
    bracket one kernel each."""
    global SERIAL
    SERIAL = bool(on)
    lib().ml_set_serial(1 if on else 0)


def timing_reset():
    lib().ml_timing_reset()


def timing_report():
    """{kernel name: (launches, total_ms)} from the library's CUDA events."""
    n = lib().ml_timing_report(None, 0)
    buf = C.create_string_buffer(int(n))
    lib().ml_timing_report(buf, n)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.rsplit(" ", 2)
        out[name] = (int(cnt), float(ms))
    return out


def _size(fn, shape):
    n = C.c_size_t(0)
    check(fn(C.byref(shape), C.byref(n)))
    return n.value


# ------------------------------------------------------------------ synth
def synth_fill(out, seed, tag, scale=1.0, cls=0, row0=0, modulus=0):
    """Counter-based generator (synthetic/gen.py semantics) into `out`
    ([rows, cols] view of a contiguous tensor; int32 for cls=3)."""
    cols = out.shape[-1] if out.dim() else 1
    rows = out.numel() // max(cols, 1)
    dt = _lib.ML_BF16 if out.dtype == torch.bfloat16 else _lib.ML_F32
    check(lib().ml_synth_fill(_p(out), rows, cols, row0, seed & (2**64 - 1), tag, scale, cls, dt,
                              modulus, _stream()))
    return out


# ------------------------------------------------------------- product keys
def pkm_shape(q, K1, k, qk_norm=False):
    T, H, Dk = q.shape
    return PkmShape(T, H, K1.shape[1], Dk, k, _dt(q), 1 if qk_norm else 0)


def pkm_topk(q, K1, K2, k, with_score=False, qk_norm=False):
    """Product-key top-k + softmax (Eq. 1).  q [T,H,Dk], K1/K2 [H,S,Dk/2].
    Returns idx [T,H,k] int32, w [T,H,k] fp32 (and pre-softmax scores)."""
    sh = pkm_shape(q, K1, k, qk_norm)
    T, H = q.shape[0], q.shape[1]
    idx = torch.empty((T, H, k), dtype=torch.int32, device=q.device)
    w = torch.empty((T, H, k), dtype=torch.float32, device=q.device)
    score = torch.empty_like(w) if with_score else None
    n = _size(lib().pkm_topk_workspace, sh)
    ws = workspace(n, q.device)
    check(lib().pkm_topk(C.byref(sh), _p(q), _p(K1), _p(K2), _p(idx), _p(w), _p(score),
                         _p(ws), n, _stream()))
    return (idx, w, score) if with_score else (idx, w)


def pkm_topk_bwd(q, K1, K2, idx, w, dw, dK1=None, dK2=None, qk_norm=False):
    """dq (overwrite) and dK1/dK2 (accumulate; zero-initialised if None)."""
    k = idx.shape[-1]
    sh = pkm_shape(q, K1, k, qk_norm)
    dq = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    if dK1 is None:
        dK1 = torch.zeros(K1.shape, dtype=torch.float32, device=q.device)
    if dK2 is None:
        dK2 = torch.zeros(K2.shape, dtype=torch.float32, device=q.device)
    n = _size(lib().pkm_topk_bwd_workspace, sh)
    ws = workspace(n, q.device)
    check(lib().pkm_topk_bwd(C.byref(sh), _p(q), _p(K1), _p(K2), _p(idx), _p(w), _p(dw),
                             _p(dq), _p(dK1), _p(dK2), _p(ws), n, _stream()))
    return dq, dK1, dK2


# ------------------------------------------------------------- EmbeddingBag
def bag_shape(V, idx, grad_dtype=torch.float32):
    return BagShape(V.shape[0], V.shape[1], idx.shape[0], idx.shape[1], _dt(V), _DT[grad_dtype])


def embbag_fwd(V, idx, w, gate_pre=None, return_ungated=False):
    """y[t] = sum_j w[t,j] V[idx[t,j]] (Eq. 1); with gate_pre: y * silu(gate_pre)."""
    sh = bag_shape(V, idx)
    y = torch.empty((idx.shape[0], V.shape[1]), dtype=V.dtype, device=V.device)
    yu = torch.empty_like(y) if (gate_pre is not None and return_ungated) else None
    check(lib().embbag_fwd(C.byref(sh), _p(V), _p(idx), _p(w), _p(gate_pre), _p(y), _p(yu),
                           _stream()))
    return (y, yu) if return_ungated else y


def _buf(bufs, name, shape, dtype, device):
    """A reusable output buffer (bufs: a caller-owned dict; None -> fresh)."""
    if bufs is None:
        return torch.empty(shape, dtype=dtype, device=device)
    t = bufs.get(name)
    if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != device:
        t = torch.empty(shape, dtype=dtype, device=device)
        bufs[name] = t
    return t


def embbag_bwd(V, idx, w, dy, sync=True, state=None, grad_dtype=torch.float32, bufs=None):
    """"reverse_indices" backward.  Returns rows [U] int32 (ascending),
    dV [U, dv] (grad_dtype: fp32, or bf16 for a bf16 table), dw [T,B] fp32
    (sync=True trims to U on the host); with sync=False returns the
    capacity-sized buffers and the device U.
    state: from embbag_bwd_prepare(N, dv, idx) (skips the sort)."""
    sh = bag_shape(V, idx, grad_dtype)
    P = idx.numel()
    rows = _buf(bufs, "rows", (P,), torch.int32, V.device)
    dV = _buf(bufs, "dV", (P, V.shape[1]), grad_dtype, V.device)
    U = _buf(bufs, "U", (1,), torch.int32, V.device)
    dw = _buf(bufs, "dw", tuple(idx.shape), torch.float32, V.device)
    n = _size(lib().embbag_bwd_workspace, sh)
    ws = workspace(n, V.device)
    if state is not None:
        check(lib().embbag_bwd_state(C.byref(sh), _p(V), _p(w), _p(dy), _p(state), state.numel(),
                                     _p(rows), _p(dV), _p(U), _p(dw), _p(ws), n, _stream()))
    else:
        check(lib().embbag_bwd(C.byref(sh), _p(V), _p(idx), _p(w), _p(dy), _p(rows), _p(dV),
                               _p(U), _p(dw), _p(ws), n, _stream()))
    if not sync:
        return rows, dV, U, dw
    u = int(U.item())
    return rows[:u], dV[:u], dw


def embbag_bwd_prepare(N, dv, idx, dtype=torch.bfloat16, out=None):
    """The inverse index map of embbag_bwd for indices idx [T,B] into an
    N-row table of width dv (include/memlayer.h embbag_bwd_prepare); returns
    the state tensor for embbag_bwd(..., state=) (`out`, if large enough, is
    reused)."""
    sh = BagShape(N, dv, idx.shape[0], idx.shape[1], _DT[dtype])
    n = _size(lib().embbag_bwd_state_bytes, sh)
    state = out if (out is not None and out.numel() >= n) else \
        torch.empty((max(n, 1),), dtype=torch.uint8, device=idx.device)
    check(lib().embbag_bwd_prepare(C.byref(sh), _p(idx), _p(state), n, _stream()))
    return state


def group_sort_local(N, idx, rank, out=None, ws=None):
    """This rank's share of the memory group's inverse map
    (include/memlayer.h embbag_bwd_group_sort_local): its positions [T_loc*B]
    sorted stably by row, tagged with global positions; returns the int32
    list [2, T_loc*B] (rows | positions)."""
    sh = BagShape(N, 8, idx.shape[0], idx.shape[1], _DT[torch.bfloat16])   # dv unused
    P = idx.numel()
    lst = out if out is not None else torch.empty((2, P), dtype=torch.int32, device=idx.device)
    n = _size(lib().embbag_bwd_group_sort_local_workspace, sh)
    ws = ws if (ws is not None and ws.numel() >= n) else workspace(n, idx.device)
    check(lib().embbag_bwd_group_sort_local(C.byref(sh), int(rank), _p(idx), _p(lst), _p(ws), n,
                                            _stream()))
    return lst


def group_merge(N, dv, lists, dtype=torch.bfloat16, out=None):
    """The G ranks' sorted lists [G, 2, T_loc*B] (rank order) -> the state of
    the bag over all G*T_loc tokens (embbag_bwd_group_merge), for
    embbag_bwd(..., state=) on the [N, dv] shard."""
    G, _, P_loc = lists.shape
    sh = BagShape(N, dv, G * P_loc, 1, _DT[dtype])
    # the state layout depends on P = T*B only: carve it as [G*P_loc, 1]
    n = _size(lib().embbag_bwd_state_bytes, sh)
    state = out if (out is not None and out.numel() >= n) else \
        torch.empty((max(n, 1),), dtype=torch.uint8, device=lists.device)
    check(lib().embbag_bwd_group_merge(C.byref(sh), int(G), _p(lists), _p(state), n, _stream()))
    return state


def embbag_bwd_dv_only(N, idx, w, dy, sync=True):
    """"reverse_indices" value gradient only (no V, no dw): rows, dV (compact)."""
    sh = BagShape(N, dy.shape[1], idx.shape[0], idx.shape[1], _dt(dy))
    P = idx.numel()
    rows = torch.empty(P, dtype=torch.int32, device=dy.device)
    dV = torch.empty((P, dy.shape[1]), dtype=torch.float32, device=dy.device)
    U = torch.empty(1, dtype=torch.int32, device=dy.device)
    n = _size(lib().embbag_bwd_workspace, sh)
    ws = workspace(n, dy.device)
    check(lib().embbag_bwd(C.byref(sh), None, _p(idx), _p(w), _p(dy), _p(rows), _p(dV), _p(U),
                           None, _p(ws), n, _stream()))
    if not sync:
        return rows, dV, U
    u = int(U.item())
    return rows[:u], dV[:u]


def embbag_bwd_atomics(N, idx, w, dy, dV_dense=None):
    """Control strategy "atomics": dense fp32 dV, accumulate."""
    sh = BagShape(N, dy.shape[1], idx.shape[0], idx.shape[1], _dt(dy))
    if dV_dense is None:
        dV_dense = torch.zeros((N, dy.shape[1]), dtype=torch.float32, device=dy.device)
    check(lib().embbag_bwd_atomics(C.byref(sh), _p(idx), _p(w), _p(dy), _p(dV_dense), _stream()))
    return dV_dense


def embbag_bwd_lock(N, idx, w, dy, dV_dense=None, locks=None):
    """Control strategy "lock": dense fp32 dV, accumulate."""
    sh = BagShape(N, dy.shape[1], idx.shape[0], idx.shape[1], _dt(dy))
    if dV_dense is None:
        dV_dense = torch.zeros((N, dy.shape[1]), dtype=torch.float32, device=dy.device)
    if locks is None:
        locks = torch.zeros(int(lib().embbag_bwd_lock_count(C.byref(sh))), dtype=torch.int32,
                            device=dy.device)
    check(lib().embbag_bwd_lock(C.byref(sh), _p(idx), _p(w), _p(dy), _p(dV_dense), _p(locks),
                                _stream()))
    return dV_dense


def sparse_adam(V, rows, dV, U, m, v, steps, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                weight_decay=0.0, V_master=None):
    """Lazy row-wise Adam(W) on the touched value rows (in place); rows/dV/U
    as returned by embbag_bwd(sync=False) or memory_layer_bwd."""
    sh = BagShape(V.shape[0], V.shape[1], rows.shape[0], 1, _dt(V), _dt(dV))
    hp = _lib.AdamParams(lr, beta1, beta2, eps, weight_decay)
    check(lib().ml_sparse_adam(C.byref(sh), _p(rows), _p(dV), _p(U), _p(V), _p(V_master), _p(m),
                               _p(v), _p(steps), C.byref(hp), _stream()))
    return V


def embbag_grad_apply(V, idx, rows, dV, U, dV_dense):
    sh = bag_shape(V, idx, dV.dtype)
    check(lib().embbag_grad_apply(C.byref(sh), _p(rows), _p(dV), _p(U), _p(dV_dense), _stream()))
    return dV_dense


# ------------------------------------------------------------ memory layer
def layer_shape(x, q, K1, V, k, gated, qk_norm=False, grad_dtype=torch.float32):
    T, H, Dk = q.shape
    D = x.shape[1] if (gated and x is not None) else V.shape[1]
    return LayerShape(PkmShape(T, H, K1.shape[1], Dk, k, _dt(q), 1 if qk_norm else 0), V.shape[0],
                      V.shape[1], D, 1 if gated else 0, _DT[grad_dtype])


def memory_layer_fwd(x, q, K1, K2, V, W1, W2, k, gated=True, qk_norm=False, keep_state=True):
    """Eq. 1 + Eq. 2 forward.  Returns out [T,D] and the saved tensors.
    keep_state: also build the backward's sorted inverse index map (a side
    stream, overlapping the bag forward) into saved["state"]."""
    sh = layer_shape(x, q, K1, V, k, gated, qk_norm)
    T, H = q.shape[0], q.shape[1]
    dev = q.device
    out = torch.empty((T, sh.D), dtype=V.dtype, device=dev)
    idx = torch.empty((T, H, k), dtype=torch.int32, device=dev)
    w = torch.empty((T, H, k), dtype=torch.float32, device=dev)
    g = torch.empty((T, V.shape[1]), dtype=V.dtype, device=dev) if gated else None
    y = torch.empty((T, V.shape[1]), dtype=V.dtype, device=dev) if gated else None
    n = _size(lib().memory_layer_fwd_workspace, sh)
    ws = workspace(n, dev)
    state, ns = None, 0
    if keep_state:
        ns = _size(lib().memory_layer_state_bytes, sh)
        state = torch.empty((max(ns, 1),), dtype=torch.uint8, device=dev)
    check(lib().memory_layer_fwd_state(C.byref(sh), _p(x if gated else None), _p(q), _p(K1),
                                       _p(K2), _p(V), _p(W1 if gated else None),
                                       _p(W2 if gated else None), _p(out), _p(idx), _p(w), _p(g),
                                       _p(y), _p(state), ns, _p(ws), n, _stream()))
    if state is not None:
        # the state is written on a library stream: before its memory can go
        # back to the caching allocator, this stream must wait for that work
        weakref.finalize(state, lib().memory_layer_state_wait, state.data_ptr(), _stream())
    return out, dict(idx=idx, w=w, g=g, y=y, k=k, gated=gated, qk_norm=qk_norm, state=state,
                     state_bytes=ns)


class LayerGrads(dict):
    __getattr__ = dict.__getitem__


def memory_layer_bwd(dout, x, q, K1, K2, V, W1, W2, saved, dK1=None, dK2=None, want_dw=False,
                     bufs=None, dV_dtype=torch.float32):
    """Backward of memory_layer_fwd.  dK1/dK2 accumulate (zeros if None).
    dV is compact: rows[:U], dV[:U] (capacity-sized buffers + device U),
    stored as dV_dtype (fp32, or bf16 for a bf16 table)."""
    k, gated = saved["k"], saved["gated"]
    sh = layer_shape(x, q, K1, V, k, gated, saved.get("qk_norm", False), dV_dtype)
    T, H = q.shape[0], q.shape[1]
    dev = q.device
    P = T * H * k
    b = bufs if bufs is not None else {}
    def buf(name, shape, dtype):
        t = b.get(name)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, device=dev)
            b[name] = t
        return t
    dq = buf("dq", q.shape, torch.float32)
    if dK1 is None:
        dK1 = torch.zeros(K1.shape, dtype=torch.float32, device=dev)
    if dK2 is None:
        dK2 = torch.zeros(K2.shape, dtype=torch.float32, device=dev)
    rows = buf("rows", (P,), torch.int32)
    dV = buf("dV", (P, V.shape[1]), dV_dtype)
    U = buf("U", (1,), torch.int32)
    dx = buf("dx", x.shape, V.dtype) if gated else None
    dW1 = buf("dW1", W1.shape, torch.float32) if gated else None
    dW2 = buf("dW2", W2.shape, torch.float32) if gated else None
    dw = buf("dw", (T, H, k), torch.float32) if want_dw else None
    n = _size(lib().memory_layer_bwd_workspace, sh)
    ws = workspace(n, dev, tag="bwd")
    check(lib().memory_layer_bwd_state(
        C.byref(sh), _p(dout), _p(x if gated else None), _p(q), _p(K1), _p(K2), _p(V),
        _p(W1 if gated else None), _p(W2 if gated else None), _p(saved["idx"]), _p(saved["w"]),
        _p(saved["g"]), _p(saved["y"]), _p(saved.get("state")), saved.get("state_bytes", 0),
        _p(dx), _p(dq), _p(dK1), _p(dK2), _p(rows), _p(dV),
        _p(U), _p(dW1), _p(dW2), _p(dw), _p(ws), n, _stream()))
    return LayerGrads(dq=dq, dK1=dK1, dK2=dK2, rows=rows, dV=dV, U=U, dx=dx, dW1=dW1, dW2=dW2,
                      dw=dw)


# ------------------------------------------------------------ PEER (f4)
def peer_shape(x, q, K1, U, k, qk_norm=False):
    T, H, Dk = q.shape
    return PeerShape(PkmShape(T, H, K1.shape[1], Dk, k, _dt(q), 1 if qk_norm else 0), U.shape[0],
                     U.shape[1])


def peer_fwd(x, q, K1, K2, U, V, k, qk_norm=False):
    """PEER-style rank-1 experts (include/memlayer.h peer_fwd).  Returns
    y [T,D] and the saved tensors (idx, w, h)."""
    sh = peer_shape(x, q, K1, U, k, qk_norm)
    T, H = q.shape[0], q.shape[1]
    dev = q.device
    y = torch.empty((T, U.shape[1]), dtype=V.dtype, device=dev)
    idx = torch.empty((T, H, k), dtype=torch.int32, device=dev)
    w = torch.empty((T, H, k), dtype=torch.float32, device=dev)
    h = torch.empty((T, H, k), dtype=torch.float32, device=dev)
    n = _size(lib().peer_fwd_workspace, sh)
    ws = workspace(n, dev)
    check(lib().peer_fwd(C.byref(sh), _p(x), _p(q), _p(K1), _p(K2), _p(U), _p(V), _p(y), _p(idx),
                         _p(w), _p(h), _p(ws), n, _stream()))
    return y, dict(idx=idx, w=w, h=h, k=k, qk_norm=qk_norm)


def peer_bwd(dy, x, q, K1, K2, U, V, saved, dK1=None, dK2=None, want_dwr=False):
    """Backward of peer_fwd: dx, dq, dK1/dK2 (accumulate), rows/dU/dV compact
    (capacity buffers + device count), dwr (router weight gradient)."""
    k = saved["k"]
    sh = peer_shape(x, q, K1, U, k, saved.get("qk_norm", False))
    T, H = q.shape[0], q.shape[1]
    dev = q.device
    P = T * H * k
    D = U.shape[1]
    dx = torch.empty_like(x)
    dq = torch.empty(q.shape, dtype=torch.float32, device=dev)
    if dK1 is None:
        dK1 = torch.zeros(K1.shape, dtype=torch.float32, device=dev)
    if dK2 is None:
        dK2 = torch.zeros(K2.shape, dtype=torch.float32, device=dev)
    rows = torch.empty((P,), dtype=torch.int32, device=dev)
    dU = torch.empty((P, D), dtype=torch.float32, device=dev)
    dV = torch.empty((P, D), dtype=torch.float32, device=dev)
    cnt = torch.empty((1,), dtype=torch.int32, device=dev)
    dwr = torch.empty((T, H, k), dtype=torch.float32, device=dev) if want_dwr else None
    n = _size(lib().peer_bwd_workspace, sh)
    ws = workspace(n, dev, tag="bwd")
    check(lib().peer_bwd(C.byref(sh), _p(dy), _p(x), _p(q), _p(K1), _p(K2), _p(U), _p(V),
                         _p(saved["idx"]), _p(saved["w"]), _p(saved["h"]), _p(dx), _p(dq),
                         _p(dK1), _p(dK2), _p(rows), _p(dU), _p(dV), _p(cnt), _p(dwr), _p(ws), n,
                         _stream()))
    return LayerGrads(dx=dx, dq=dq, dK1=dK1, dK2=dK2, rows=rows, dU=dU, dV=dV, U=cnt, dwr=dwr)


# ------------------------------------------------------- group / gate pieces
def group_unpack(recv, G, T_loc, dv, gate=None, want_y=True):
    """recv [G, T_loc, dv/G] -> y [T_loc, dv] (and z = y*silu(gate) if gate)."""
    dt = _dt(recv)
    y = torch.empty((T_loc, dv), dtype=recv.dtype, device=recv.device) if want_y else None
    z = torch.empty((T_loc, dv), dtype=recv.dtype, device=recv.device) if gate is not None else None
    check(lib().ml_group_unpack(_p(recv), G, T_loc, dv, _p(gate), _p(y), _p(z), dt, _stream()))
    return y, z


def group_pack(src, G):
    """src [T_loc, dv] -> [G, T_loc, dv/G] (slice g of every token row)."""
    T_loc, dv = src.shape
    dst = torch.empty((G, T_loc, dv // G), dtype=src.dtype, device=src.device)
    check(lib().ml_group_pack(_p(src), G, T_loc, dv, _p(dst), _dt(src), _stream()))
    return dst


def gate_bwd(dz, g, y):
    """Eq. 2 elementwise backward: returns z = y*silu(g), dy, dg."""
    z, dy, dg = torch.empty_like(y), torch.empty_like(y), torch.empty_like(y)
    check(lib().ml_gate_bwd(_p(dz), _p(g), _p(y), _p(z), _p(dy), _p(dg), y.numel(), _dt(y),
                            _stream()))
    return z, dy, dg


def gemm(A, B, transA=False, transB=False, out_f32=False):
    """Row-major C = op(A) op(B) on cuBLASLt (library GEMM)."""
    M = A.shape[1] if transA else A.shape[0]
    K = A.shape[0] if transA else A.shape[1]
    N = B.shape[0] if transB else B.shape[1]
    C_ = torch.empty((M, N), dtype=torch.float32 if out_f32 else A.dtype, device=A.device)
    ws = workspace(32 << 20, A.device, tag="gemm")
    check(lib().ml_gemm(1 if transA else 0, 1 if transB else 0, M, N, K, _p(A), A.shape[1], _p(B),
                        B.shape[1], _p(C_), N, _dt(A), 1 if out_f32 else 0, _p(ws), ws.numel(),
                        _stream()))
    return C_


def embbag_bwd_pool(V, idx_list, w_list, dy_list):
    """Shared memory pool (one (K, V) pool for all memory layers;
    SURVEY f1): the value gradient of L layers in ONE sort and ONE segmented
    pass.  The layers' positions are concatenated (token-major), so a row hit
    by several layers is reduced once; returns rows, dV, U (capacity-sized,
    device U) and the per-layer dw."""
    idx = torch.cat(idx_list, 0)
    w = torch.cat(w_list, 0)
    dy = torch.cat(dy_list, 0)
    rows, dV, U, dw = embbag_bwd(V, idx, w, dy, sync=False)
    return rows, dV, U, list(torch.split(dw, [i.shape[0] for i in idx_list], 0))


# ------------------------------------------------------------ device guard
def _on_device(fn):
    """Run `fn` with the device of its first CUDA tensor argument current, so
    the library launches on that device and on that device's current stream
    (tensors on a non-current device otherwise get the wrong stream)."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        for a in list(args) + list(kwargs.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                if a.device.index == torch.cuda.current_device():
                    return fn(*args, **kwargs)
                with torch.cuda.device(a.device):
                    return fn(*args, **kwargs)
        return fn(*args, **kwargs)
    return wrapped


for _name in ("synth_fill", "pkm_topk", "pkm_topk_bwd", "embbag_fwd", "embbag_bwd",
              "embbag_bwd_prepare", "embbag_bwd_dv_only", "embbag_bwd_atomics", "embbag_bwd_lock",
              "sparse_adam", "embbag_grad_apply", "memory_layer_fwd", "memory_layer_bwd", "peer_fwd",
              "peer_bwd", "group_unpack", "group_pack", "gate_bwd", "gemm", "embbag_bwd_pool"):
    globals()[_name] = _on_device(globals()[_name])
del _name


# ------------------------------------------------------------ memory group (C ABI)
MODES = {"alltoall": 0, "allgather": 1}


class Group:
    """A memory group handle (include/memlayer.h mlGroup): NCCL (one process
    per GPU; `unique_id` from group_unique_id() on one rank, broadcast by the
    caller) or an in-process hub (G ranks as host threads on one device)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        G, r = C.c_int(), C.c_int()
        check(lib().ml_group_info(self.h, C.byref(G), C.byref(r)))
        self.size, self.rank = G.value, r.value

    @classmethod
    def nccl(cls, unique_id, G, rank):
        out = C.c_void_p()
        check(lib().ml_group_init(C.c_char_p(bytes(unique_id)), G, rank, C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_hub(cls, hub, rank):
        out = C.c_void_p()
        check(lib().ml_group_init_hub(C.c_void_p(hub), rank, C.byref(out)))
        return cls(out.value)

    @classmethod
    def loopback(cls, G, rank, captures=()):
        """One rank of a G-rank group with the network removed
        (ml_group_init_loopback): `captures` are device tensors (kept alive by
        the group object) the all-gathers take the other ranks' chunks from."""
        caps = [c.contiguous() for c in captures]
        n = len(caps)
        ptrs = (C.c_void_p * max(n, 1))(*[c.data_ptr() for c in caps])
        sizes = (C.c_size_t * max(n, 1))(*[c.numel() * c.element_size() for c in caps])
        out = C.c_void_p()
        check(lib().ml_group_init_loopback(G, rank, ptrs, sizes, n, C.byref(out)))
        g = cls(out.value)
        g._captures = caps
        return g

    def set_p2p(self, on=True):
        """The fused peer-memory forward exchange (ml_group_set_p2p); every
        rank of the group must make the same choice."""
        check(lib().ml_group_set_p2p(self.h, 1 if on else 0))
        return self

    def close(self):
        if self.h:
            check(lib().ml_group_destroy(self.h))
            self.h = None


def group_unique_id():
    buf = C.create_string_buffer(128)
    check(lib().ml_group_unique_id(buf))
    return buf.raw


def group_hub(G):
    out = C.c_void_p()
    check(lib().ml_group_hub_create(G, C.byref(out)))
    return out.value


def group_hub_destroy(hub):
    lib().ml_group_hub_destroy(C.c_void_p(hub))


def memory_layer_fwd_group(grp, x, q, K1, K2, V_shard, W1, W2, k, mode="alltoall", keep_state=True,
                           bufs=None):
    """Eq. 1 + Eq. 2 over a dim-sharded memory group (§3.1.2):
    x/q of this rank's T_loc tokens, V_shard [N, dv/G].  Returns out [T_loc, D]
    and the saved tensors (idx/w of own and all tokens, g, y, y_all, state).
    bufs (a caller-owned dict): outputs and saved tensors reused across calls
    (valid until the next forward with the same dict)."""
    G = grp.size
    T, H, Dk = q.shape
    dv = V_shard.shape[1] * G
    sh = LayerShape(PkmShape(T, H, K1.shape[1], Dk, k, _dt(q), 0), V_shard.shape[0], dv, x.shape[1],
                    1, _lib.ML_F32)
    dev = q.device
    md = MODES[mode]
    out = _buf(bufs, "out", (T, x.shape[1]), q.dtype, dev)
    idx = _buf(bufs, "idx", (T, H, k), torch.int32, dev)
    w = _buf(bufs, "w", (T, H, k), torch.float32, dev)
    idx_all = _buf(bufs, "idx_all", (G * T, H, k), torch.int32, dev)
    w_all = _buf(bufs, "w_all", (G * T, H, k), torch.float32, dev)
    g = _buf(bufs, "g", (T, dv), q.dtype, dev)
    y = _buf(bufs, "y", (T, dv), q.dtype, dev)
    y_all = _buf(bufs, "y_all", (G * T, dv), q.dtype, dev) if md == 1 else None
    state, nst = None, 0
    if keep_state:
        bs = BagShape(V_shard.shape[0], dv, T, H * k, _dt(q), _lib.ML_F32)
        nst = _size(lambda b, p: lib().embbag_bwd_group_state_bytes(grp.h, b, p), bs)
        state = _buf(bufs, "state", (max(nst, 1),), torch.uint8, dev)
    n = _size(lambda b, p: lib().memory_layer_fwd_group_workspace(grp.h, b, md, p), sh)
    ws = workspace(n, dev, tag="group_fwd")
    check(lib().memory_layer_fwd_group(grp.h, C.byref(sh), md, _p(x), _p(q), _p(K1), _p(K2),
                                       _p(V_shard), _p(W1), _p(W2), _p(out), _p(idx), _p(w),
                                       _p(idx_all), _p(w_all), _p(g), _p(y), _p(y_all), _p(state),
                                       nst, _p(ws), n, _stream()))
    return out, dict(idx=idx, w=w, idx_all=idx_all, w_all=w_all, g=g, y=y, y_all=y_all, k=k,
                     state=state, state_bytes=nst, mode=mode)


def memory_layer_bwd_group(grp, dout, x, q, K1, K2, V_shard, W1, W2, saved, dK1=None, dK2=None,
                           dV_dtype=torch.float32, want_dw=False, bufs=None):
    """Backward of memory_layer_fwd_group: dx, dq, dK1/dK2 (accumulate; this
    rank's tokens' part), compact dV of the shard (rows[:U], dV[:U]), dW1,
    dW2 (this rank's part), dw of own tokens (want_dw)."""
    G = grp.size
    T, H, Dk = q.shape
    k = saved["k"]
    dv = V_shard.shape[1] * G
    sh = LayerShape(PkmShape(T, H, K1.shape[1], Dk, k, _dt(q), 0), V_shard.shape[0], dv, x.shape[1],
                    1, _DT[dV_dtype])
    dev = q.device
    P = G * T * H * k
    dx = _buf(bufs, "dx", tuple(x.shape), x.dtype, dev)
    dq = _buf(bufs, "dq", tuple(q.shape), torch.float32, dev)
    if dK1 is None:
        dK1 = torch.zeros(K1.shape, dtype=torch.float32, device=dev)
    if dK2 is None:
        dK2 = torch.zeros(K2.shape, dtype=torch.float32, device=dev)
    rows = _buf(bufs, "rows", (P,), torch.int32, dev)
    dV = _buf(bufs, "dV", (P, V_shard.shape[1]), dV_dtype, dev)
    U = _buf(bufs, "U", (1,), torch.int32, dev)
    dW1 = _buf(bufs, "dW1", tuple(W1.shape), torch.float32, dev)
    dW2 = _buf(bufs, "dW2", tuple(W2.shape), torch.float32, dev)
    dw = _buf(bufs, "dw", (T, H, k), torch.float32, dev) if want_dw else None
    n = _size(lambda b, p: lib().memory_layer_bwd_group_workspace(grp.h, b, p), sh)
    ws = workspace(n, dev, tag="group_bwd")
    check(lib().memory_layer_bwd_group(
        grp.h, C.byref(sh), _p(dout), _p(x), _p(q), _p(K1), _p(K2), _p(V_shard), _p(W1), _p(W2),
        _p(saved["idx"]), _p(saved["w"]), _p(saved["idx_all"]), _p(saved["w_all"]), _p(saved["g"]),
        _p(saved["y"]), _p(saved["state"]), saved["state_bytes"], _p(dx), _p(dq), _p(dK1), _p(dK2),
        _p(rows), _p(dV), _p(U), _p(dW1), _p(dW2), _p(dw), _p(ws), n, _stream()))
    return LayerGrads(dx=dx, dq=dq, dK1=dK1, dK2=dK2, rows=rows, dV=dV, U=U, dW1=dW1, dW2=dW2, dw=dw)


def embbag_fwd_group(grp, V_shard, idx, w, mode="alltoall"):
    """Bag level: returns y (alltoall: [T_loc, dv]; allgather: [G*T_loc, dv]),
    idx_all, w_all [G*T_loc, B]."""
    G = grp.size
    T, B = idx.shape
    dv = V_shard.shape[1] * G
    sh = BagShape(V_shard.shape[0], dv, T, B, _dt(V_shard), _lib.ML_F32)
    md = MODES[mode]
    y = torch.empty(((G if md == 1 else 1) * T, dv), dtype=V_shard.dtype, device=V_shard.device)
    idx_all = torch.empty((G * T, B), dtype=torch.int32, device=V_shard.device)
    w_all = torch.empty((G * T, B), dtype=torch.float32, device=V_shard.device)
    n = _size(lambda b, p: lib().embbag_fwd_group_workspace(grp.h, b, md, p), sh)
    ws = workspace(n, V_shard.device, tag="group_fwd")
    check(lib().embbag_fwd_group(grp.h, C.byref(sh), _p(V_shard), _p(idx), _p(w), _p(idx_all),
                                 _p(w_all), md, _p(y), _p(ws), n, _stream()))
    return y, idx_all, w_all


def embbag_bwd_group(grp, V_shard, idx_all, w_all, dy, mode="alltoall", grad_dtype=torch.float32):
    """Bag level backward: rows, dV_shard (capacity), device U, dw_local [T_loc, B]."""
    G = grp.size
    TG, B = idx_all.shape
    T = TG // G
    dv = V_shard.shape[1] * G
    sh = BagShape(V_shard.shape[0], dv, T, B, _dt(V_shard), _DT[grad_dtype])
    md = MODES[mode]
    rows = torch.empty(TG * B, dtype=torch.int32, device=V_shard.device)
    dV = torch.empty((TG * B, V_shard.shape[1]), dtype=grad_dtype, device=V_shard.device)
    U = torch.empty(1, dtype=torch.int32, device=V_shard.device)
    dw = torch.empty((T, B), dtype=torch.float32, device=V_shard.device)
    n = _size(lambda b, p: lib().embbag_bwd_group_workspace(grp.h, b, md, p), sh)
    ws = workspace(n, V_shard.device, tag="group_bwd")
    check(lib().embbag_bwd_group(grp.h, C.byref(sh), _p(V_shard), _p(idx_all), _p(w_all), _p(dy),
                                 md, None, 0, _p(rows), _p(dV), _p(U), _p(dw), _p(ws), n, _stream()))
    return rows, dV, U, dw


for _name in ("memory_layer_fwd_group", "memory_layer_bwd_group", "embbag_fwd_group",
              "embbag_bwd_group"):
    globals()[_name] = _on_device(globals()[_name])
del _name
