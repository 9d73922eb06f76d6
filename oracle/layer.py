"""The memory layer: Eq. 1 lookup + the Memory+ gate of Eq. 2
(P:189), forward and backward, composed from pkm / bag / gate.

The query q is an input (reading Q11: the query projection is outside the
hot path); dx returned by the backward is the gate-path part only.
"""
import numpy as np

from . import pkm, bag, gate


def memory_layer_fwd(x, q, K1, K2, V, W1, W2, k, gated=True, method="two_stage", qk_norm=False):
    T, H, _ = q.shape
    idx, score, w = pkm.pkm_lookup(q, K1, K2, k, method=method, qk_norm=qk_norm)
    bidx = idx.reshape(T, H * k)
    bw = w.reshape(T, H * k)
    y = bag.embbag_fwd(V, bidx, bw)
    saved = dict(idx=idx, score=score, w=w, y=y, qk_norm=qk_norm)
    if not gated:
        return y, saved
    out, g, z = gate.gate_fwd(x, y, W1, W2)
    saved.update(g=g, z=z)
    return out, saved


def memory_layer_bwd(dout, x, q, K1, K2, V, W1, W2, saved, gated=True):
    T, H, k = saved["idx"].shape
    grads = {}
    if gated:
        gb = gate.gate_bwd(dout, x, saved["y"], saved["g"], W1, W2)
        dy = gb["dy"]
        grads.update(dx=gb["dx"], dW1=gb["dW1"], dW2=gb["dW2"])
    else:
        dy = np.asarray(dout, np.float64)
    bidx = saved["idx"].reshape(T, H * k)
    bw = saved["w"].reshape(T, H * k)
    rows, dV, dw = bag.embbag_bwd(V, bidx, bw, dy)
    dq, dK1, dK2, ds = pkm.pkm_bwd(q, K1, K2, saved["idx"], saved["w"],
                                  dw.reshape(T, H, k), qk_norm=saved.get("qk_norm", False))
    grads.update(dy=dy, rows=rows, dV=dV, dw=dw.reshape(T, H, k), dq=dq,
                 dK1=dK1, dK2=dK2)
    return grads
