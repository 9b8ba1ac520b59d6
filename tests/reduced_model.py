"""numpy model of the B200 algorithm (reduced-coordinate Sherman-Morrison):
Gram pass -> N levels on the N x 2N Gram -> A, T, Z.  Test infrastructure:
used to check the algebra on CPU and to stand in for the device stages in the
gloo multi-rank test of the sharded orchestration."""

import numpy as np

SINGULAR_TOL = 1e-14


class ModelSingular(ArithmeticError):
    def __init__(self, level, den):
        self.level, self.denominator = level, den
        super().__init__(f"level {level} singular ({den})")


def gram_analysis(x_rows, y_rows, r):
    """Level-0 Gram of gathered rows: [V'R^-1 V | V'R^-1 D] with V = (x - mean)/sqrt(N-1)."""
    n = x_rows.shape[1]
    s = x_rows - x_rows.mean(axis=1, keepdims=True)
    d = y_rows - x_rows
    w = s / r[:, None]
    return np.concatenate([(w.T @ s) / (n - 1), (w.T @ d) / np.sqrt(n - 1)], axis=1)


def gram_solve(v, d, r):
    w = v / r[:, None]
    return np.concatenate([w.T @ v, w.T @ d], axis=1)


def levels(gram):
    """The N Sherman-Morrison levels on the Gram; returns (A, den)."""
    g = np.array(gram, dtype=float)
    n = g.shape[0]
    den = np.empty(n)
    for k in range(n):
        dk = 1.0 + g[k, k]
        if abs(dk) < SINGULAR_TOL:
            raise ModelSingular(k + 1, dk)
        den[k] = dk
        q = g[k, k + 1:] / dk
        g[:, k + 1:] -= np.outer(g[:, k], q)
    return g[:, n:].copy(), den


def transform(a):
    n = a.shape[0]
    return np.eye(n) + (a - a.mean(axis=0, keepdims=True)) / np.sqrt(n - 1)


def analysis(x, y, idx, r):
    xo = x if idx is None else x[idx]
    a, _ = levels(gram_analysis(xo, y, r))
    return x @ transform(a)


def solve(r, v, d):
    a, _ = levels(gram_solve(v, d, r))
    return (d - v @ a) / r[:, None], a
