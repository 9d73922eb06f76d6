"""PyTorch autograd wrapper over the C-ABI memory layer (argument marshalling
only: every step of the forward and backward runs in libmemlayer kernels).

    y = MemoryLayerFunction.apply(x, q, K1, K2, V, W1, W2, k, qk_norm)

is Eq. 1 + Eq. 2 of PAPER.md (P:148-149 product-key lookup + EmbeddingBag,
P:189 Memory+ silu gate): forward = `memory_layer_fwd` (with the backward's
sorted inverse index map built on a side stream), backward =
`memory_layer_bwd`.  The value-table gradient is returned SPARSE (a COO
tensor over the touched rows, "reverse_indices": dV exists only for the
distinct rows a step touched), as nn.Embedding(sparse=True) does; pass
`dense_value_grad=True` to MemoryLayer for a dense gradient instead.

`MemoryLayer` is the module form: the query projection (a plain torch GEMM,
outside the hot path), the per-head half-key tables K1, K2 [H, S, Dk/2], the
values V [S*S, dv] and the gate weights W1 [D, dv], W2 [dv, D].
"""
import math

import torch

from . import ops


class MemoryLayerFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, q, K1, K2, V, W1, W2, k, qk_norm=False, dense_value_grad=False):
        x, q = x.contiguous(), q.contiguous()
        # the library launches on the current device's current stream: make
        # the inputs' device current (a layer on cuda:1 without set_device)
        with torch.cuda.device(x.device):
            out, saved = ops.memory_layer_fwd(x, q, K1, K2, V, W1, W2, k, gated=True,
                                              qk_norm=qk_norm, keep_state=True)
        ctx.saved = saved
        ctx.dense_value_grad = dense_value_grad
        ctx.save_for_backward(x, q, K1, K2, V, W1, W2)
        return out

    @staticmethod
    def backward(ctx, dout):
        x, q, K1, K2, V, W1, W2 = ctx.saved_tensors
        with torch.cuda.device(x.device):
            g = ops.memory_layer_bwd(dout.contiguous().to(V.dtype), x, q, K1, K2, V, W1, W2,
                                     ctx.saved)
        U = int(g.U.item())
        rows = g.rows[:U].long()
        if ctx.dense_value_grad:
            dV = torch.zeros(V.shape, dtype=torch.float32, device=V.device)
            if U:
                dV[rows] = g.dV[:U]                   # rows are distinct
            dV = dV.to(V.dtype)
        else:
            dV = torch.sparse_coo_tensor(rows.unsqueeze(0), g.dV[:U].to(V.dtype), V.shape,
                                         is_coalesced=True, check_invariants=False)
        ctx.saved = None
        return (g.dx, g.dq.to(q.dtype), g.dK1.to(K1.dtype), g.dK2.to(K2.dtype), dV,
                g.dW1.to(W1.dtype), g.dW2.to(W2.dtype), None, None, None)


class MemoryLayer(torch.nn.Module):
    """Memory+ layer (Eq. 1-2) over S*S product keys.

    D: model dim, dv: value dim, H: heads, S: sub-keys per half (N = S*S
    values), Dk: query/key dim per head, k: keys per head.  Inputs [..., D]."""

    def __init__(self, D, dv, H=4, S=1024, Dk=None, k=32, qk_norm=False, dense_value_grad=False,
                 dtype=torch.bfloat16, device=None):
        super().__init__()
        Dk = Dk if Dk is not None else dv // 2           # reading Q3: Dk = dv / 2
        self.D, self.dv, self.H, self.S, self.Dk, self.k = D, dv, H, S, Dk, k
        self.qk_norm, self.dense_value_grad = qk_norm, dense_value_grad
        f = dict(dtype=dtype, device=device)
        self.query = torch.nn.Linear(D, H * Dk, bias=False, **f)
        self.K1 = torch.nn.Parameter(torch.randn(H, S, Dk // 2, **f) / math.sqrt(Dk // 2))
        self.K2 = torch.nn.Parameter(torch.randn(H, S, Dk // 2, **f) / math.sqrt(Dk // 2))
        self.V = torch.nn.Parameter(torch.randn(S * S, dv, **f) / math.sqrt(dv))
        self.W1 = torch.nn.Parameter(torch.randn(D, dv, **f) / math.sqrt(D))
        self.W2 = torch.nn.Parameter(torch.randn(dv, D, **f) / math.sqrt(dv))

    def forward(self, x):
        shape = x.shape
        x2 = x.reshape(-1, self.D)
        q = self.query(x2).reshape(-1, self.H, self.Dk)
        y = MemoryLayerFunction.apply(x2, q, self.K1, self.K2, self.V, self.W1, self.W2, self.k,
                                      self.qk_norm, self.dense_value_grad)
        return y.reshape(*shape[:-1], self.D)
