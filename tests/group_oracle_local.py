"""CPU local-compute backend for paper_2412_09764_b200.group built from the
oracle (test infrastructure): lets the memory-group protocol run under
torch.distributed gloo on CPU with world size 2."""
import numpy as np
import torch

from oracle import bag as obag, gate as ogate, pkm as opkm


def _np(t):
    return t.detach().cpu().numpy()


class OracleLocal:
    grad_dtype = torch.float64

    def empty(self, shape, dtype, like):
        return torch.empty(shape, dtype=dtype)

    def pkm_topk(self, q, K1, K2, k):
        idx, score, w = opkm.pkm_lookup(_np(q), _np(K1), _np(K2), k)
        return torch.from_numpy(idx.astype(np.int32)), torch.from_numpy(w)

    def embbag_fwd(self, V, idx, w):
        return torch.from_numpy(obag.embbag_fwd(_np(V), _np(idx), _np(w)))

    def embbag_bwd(self, V, idx, w, dy):
        rows, dV, dw = obag.embbag_bwd(_np(V), _np(idx), _np(w), _np(dy))
        return (torch.from_numpy(rows.astype(np.int32)), torch.from_numpy(dV),
                torch.tensor([rows.size], dtype=torch.int32), torch.from_numpy(dw))

    def pkm_topk_bwd(self, q, K1, K2, idx, w, dw, dK1, dK2):
        dq, a, b, _ = opkm.pkm_bwd(_np(q), _np(K1), _np(K2), _np(idx).astype(np.int64), _np(w), _np(dw))
        dK1 += torch.from_numpy(a)
        dK2 += torch.from_numpy(b)
        return torch.from_numpy(dq), dK1, dK2

    def gemm(self, A, B, transA=False, transB=False, out_f32=False):
        a = _np(A).T if transA else _np(A)
        b = _np(B).T if transB else _np(B)
        return torch.from_numpy(a @ b)

    def unpack(self, recv, G, T_loc, dv, gate=None, want_y=True):
        r = _np(recv)                                   # [G, T_loc, dv/G]
        y = np.concatenate([r[g] for g in range(G)], axis=1)
        z = y * ogate.silu(_np(gate)) if gate is not None else None
        return (torch.from_numpy(y) if want_y else None,
                torch.from_numpy(z) if z is not None else None)

    def pack(self, src, G):
        s = _np(src)
        T_loc, dv = s.shape
        return torch.from_numpy(np.ascontiguousarray(s.reshape(T_loc, G, dv // G).transpose(1, 0, 2)))

    def gate_bwd(self, dz, g, y):
        dz, g, y = _np(dz), _np(g), _np(y)
        z = y * ogate.silu(g)
        return torch.from_numpy(z), torch.from_numpy(dz * ogate.silu(g)), \
            torch.from_numpy(dz * y * ogate.dsilu(g))
