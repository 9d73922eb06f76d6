"""Memory+ gating, Eq. 2 (Fig. 3):

    output = (y ⊙ silu(x^T W1))^T W2,   silu(x) = x sigmoid(x)

Reading Q10: with row-vector tokens, g = x W1 (W1 in R^{D x dv}),
z = y ⊙ silu(g), out = z W2 (W2 in R^{dv x D}).  float64.
"""
import numpy as np


def sigmoid(x):
    x = np.asarray(x, np.float64)
    return np.where(x >= 0, 1.0 / (1.0 + np.exp(-np.abs(x))),
                    np.exp(-np.abs(x)) / (1.0 + np.exp(-np.abs(x))))


def silu(x):
    """silu(x) = x sigmoid(x)."""
    return np.asarray(x, np.float64) * sigmoid(x)


def dsilu(x):
    """d/dx [x sigmoid(x)] = sigmoid(x) (1 + x (1 - sigmoid(x)))."""
    s = sigmoid(x)
    return s * (1.0 + np.asarray(x, np.float64) * (1.0 - s))


def gate_fwd(x, y, W1, W2):
    """Eq. 2 forward.  Returns out [T, D], g = x W1 [T, dv], z [T, dv]."""
    g = np.asarray(x, np.float64) @ np.asarray(W1, np.float64)
    z = np.asarray(y, np.float64) * silu(g)
    return z @ np.asarray(W2, np.float64), g, z


def gate_bwd(dout, x, y, g, W1, W2):
    """Eq. 2 backward (chain rule):
    dz = dout W2^T, dW2 = z^T dout, dy = dz ⊙ silu(g),
    dg = dz ⊙ y ⊙ silu'(g), dW1 = x^T dg, dx = dg W1^T."""
    dout = np.asarray(dout, np.float64)
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    W1 = np.asarray(W1, np.float64)
    W2 = np.asarray(W2, np.float64)
    z = y * silu(g)
    dz = dout @ W2.T
    dW2 = z.T @ dout
    dy = dz * silu(g)
    dg = dz * y * dsilu(g)
    dW1 = x.T @ dg
    dx = dg @ W1.T
    return dict(dy=dy, dx=dx, dW1=dW1, dW2=dW2, dz=dz, dg=dg)
