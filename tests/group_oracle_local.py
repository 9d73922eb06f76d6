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

    # the group's inverse map (include/memlayer.h embbag_bwd_group_sort_local
    # / _merge): own positions stably sorted by row with global positions,
    # then a G-way merge of the gathered lists (ties to the lower rank)
    def group_sort_local(self, N, idx, rank):
        flat = _np(idx).reshape(-1).astype(np.int64)
        order = np.argsort(flat, kind="stable")
        return torch.from_numpy(np.stack([flat[order], order + rank * flat.size]).astype(np.int32))

    def group_lists(self, G, lst):
        return torch.empty((G,) + tuple(lst.shape), dtype=lst.dtype)

    def group_merge(self, N, dv, lists, dtype):
        import heapq
        L = _np(lists)
        runs = [[(int(L[g, 0, i]), g, int(L[g, 1, i])) for i in range(L.shape[2])] for g in range(L.shape[0])]
        merged = list(heapq.merge(*runs, key=lambda e: (e[0], e[1])))
        return np.array([[e[0] for e in merged], [e[2] for e in merged]], dtype=np.int64), None

    def wait(self, ev):
        pass

    def embbag_bwd(self, V, idx, w, dy, state=None):
        if state is not None:    # the merged map is the stable sort of all gathered positions
            flat = _np(idx).reshape(-1).astype(np.int64)
            order = np.argsort(flat, kind="stable")
            assert np.array_equal(state[1], order) and np.array_equal(state[0], flat[order])
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
