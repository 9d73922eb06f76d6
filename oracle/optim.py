"""Sparse (lazy, row-wise) Adam for the memory values (SPEC.md
S:472-476 OptimizerState / S:506-514 sparse_adam_update).

PAPER.md P:167 only names the problem ("the large number of trainable
parameters and associated optimizer states"); the update rule follows SPEC:
Adam applied only to the touched value rows, with per-row step counters for
the bias correction; untouched rows unchanged.  Decoupled weight decay
(AdamW form) is optional.  float64.
"""
import numpy as np


def sparse_adam_step(V, m, v, steps, rows, dV, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                     weight_decay=0.0):
    """In place on V [N, dv], m, v [N, dv], steps [N] for the rows `rows`
    (distinct) with gradients dV [len(rows), dv]:
        c = ++steps[r]
        m[r] = beta1 m[r] + (1 - beta1) g
        v[r] = beta2 v[r] + (1 - beta2) g^2
        V[r] -= lr * ( (m[r] / (1 - beta1^c)) / (sqrt(v[r] / (1 - beta2^c)) + eps)
                       + weight_decay * V[r] )
    """
    rows = np.asarray(rows, np.int64)
    for i, r in enumerate(rows):
        g = np.asarray(dV[i], np.float64)
        steps[r] += 1
        c = steps[r]
        m[r] = beta1 * m[r] + (1.0 - beta1) * g
        v[r] = beta2 * v[r] + (1.0 - beta2) * g * g
        mhat = m[r] / (1.0 - beta1 ** c)
        vhat = v[r] / (1.0 - beta2 ** c)
        V[r] = V[r] - lr * (mhat / (np.sqrt(vhat) + eps) + weight_decay * V[r])


def dense_adam_step(V, m, v, step, dV_dense, lr, beta1=0.9, beta2=0.999, eps=1e-8,
                    weight_decay=0.0):
    """Textbook dense Adam(W) on the whole table with one global step count
    (the pin: equals sparse_adam_step when every row is touched every step)."""
    g = np.asarray(dV_dense, np.float64)
    m[:] = beta1 * m + (1.0 - beta1) * g
    v[:] = beta2 * v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** step)
    vhat = v / (1.0 - beta2 ** step)
    V[:] = V - lr * (mhat / (np.sqrt(vhat) + eps) + weight_decay * V)
