"""numpy/scipy restatement of the reference analysis path (TEST INFRASTRUCTURE).

Each function cites the reference lines it restates.  The BLAS call sequence
of the grouped sweep (ddot/dgemv, dger, dgemm with overwrite) is kept so that,
on the same host and BLAS build, the restatement reproduces the reference's
rounding; across hosts it agrees to BLAS-kernel rounding (~1e-15 relative).

Reference files (read-only, not shipped):
  enkf.py    = /root/reference/pkg/src/enkfkit/enkf.py
  sherman.py = /root/reference/pkg/src/enkfkit/sherman.py
"""

from __future__ import annotations

import numpy as np
from scipy.linalg.blas import dgemm, dger

# sherman.py:51 — guard on |1 + v'u|
SINGULAR_TOL = 1e-14
# sherman.py:146 — levels per compound trailing update
GROUP_LEVELS = 8


class OracleSingularUpdate(ArithmeticError):
    """Oracle-side twin of `SingularUpdateError(level, denominator)`
    (errors.py:15-29): ``level`` is 1-based."""

    def __init__(self, level: int, denominator: float):
        self.level = level
        self.denominator = denominator
        super().__init__(f"rank-one update {level} singular (1 + v'u = {denominator:.3e})")


def long_op_count(nens: int, nobs: int) -> int:
    """sherman.py:73-82 — 3 (N^2 Nobs + N Nobs) multiplications/divisions."""
    if nens < 1 or nobs < 1:
        raise ValueError("nens and nobs must be at least 1")
    return 3 * nobs * nens * (nens + 1)


def member_deviations(x):
    """enkf.py:82-92 — S = (X - row mean) / sqrt(N - 1); N >= 2."""
    ens = np.asarray(x, dtype=float)
    if ens.ndim != 2 or ens.shape[1] < 2:
        raise ValueError("need at least 2 ensemble members for deviations")
    centre = ens.mean(axis=1, keepdims=True)
    return (ens - centre) / np.sqrt(ens.shape[1] - 1.0)


def apply_selection(indices, x):
    """enkf.py:50-59 — row gather by sorted indices; None = identity (alias)."""
    if indices is None:
        return x
    if indices[-1] >= x.shape[0]:
        raise IndexError(f"observation index {indices[-1]} out of range for state size {x.shape[0]}")
    return x[indices]


def innovations(perturbed, indices, x):
    """enkf.py:114-120 — D = Y - H(X)."""
    return perturbed - apply_selection(indices, np.asarray(x, dtype=float))


def validate_system(r, v, d):
    """sherman.py:85-108 — shape, positivity and finiteness checks."""
    r, v, d = (np.asarray(a, dtype=float) for a in (r, v, d))
    if r.ndim != 1:
        raise ValueError(f"r must be a vector, got shape {r.shape}")
    if v.ndim != 2 or d.ndim != 2:
        raise ValueError("V and D must be matrices")
    n = r.shape[0]
    if v.shape[0] != n or d.shape[0] != n:
        raise ValueError(f"row mismatch: r {n}, V {v.shape[0]}, D {d.shape[0]}")
    if v.shape[1] != d.shape[1]:
        raise ValueError(f"column mismatch: V {v.shape[1]}, D {d.shape[1]}")
    if v.shape[1] < 1:
        raise ValueError("need at least one ensemble column")
    if np.any(r <= 0):
        raise ValueError("observation variances must be positive")
    if not (np.isfinite(v).all() and np.isfinite(d).all() and np.isfinite(r).all()):
        raise ValueError("inputs contain non-finite entries")
    return r, v, d


def _level0_panel(r, v, d):
    """sherman.py:149-154 — level 0 G = [V/r | D/r], Fortran order."""
    nobs, nens = v.shape
    panel = np.empty((nobs, 2 * nens), order="F")
    np.divide(v, r[:, None], out=panel[:, :nens])
    np.divide(d, r[:, None], out=panel[:, nens:])
    return panel


def _checked_denominator(vk, u, level):
    den = 1.0 + float(vk @ u)
    if abs(den) < SINGULAR_TOL:
        raise OracleSingularUpdate(level, den)
    return den


def sweep_grouped(r, v, d, group=GROUP_LEVELS):
    """sherman.py:157-214 (workers=1) — the production grouped sweep.

    For each group of `group` pivot levels: build h_j = u_j / den_j and the
    lower-triangular composition C (sherman.py:167-187, eager dger on the
    group's later pivots), then one compound update of the trailing columns
    G_trail -= H (C (V_blk' G_trail)) (sherman.py:208-214).  Returns Z (C order).
    """
    nobs, nens = v.shape
    panel = _level0_panel(r, v, d)
    for k0 in range(0, nens, group):
        width = min(group, nens - k0)
        hcols = np.empty((nobs, width), order="F")
        comp = np.zeros((width, width))
        for j in range(width):
            lvl = k0 + j
            vk = v[:, lvl]
            den = _checked_denominator(vk, panel[:, lvl], lvl + 1)
            h = panel[:, lvl] / den
            hcols[:, j] = h
            if j:
                comp[j, :j] = -((vk @ hcols[:, :j]) @ comp[:j, :j])
            comp[j, j] = 1.0
            if j + 1 < width:
                pivots = panel[:, lvl + 1:k0 + width]
                dger(-1.0, h, vk @ pivots, a=pivots, overwrite_a=1)
        lo = k0 + width
        if lo < 2 * nens:
            trailing = panel[:, lo:]
            coef = comp @ (v[:, k0:k0 + width].T @ trailing)
            dgemm(-1.0, hcols, coef, beta=1.0, c=trailing, overwrite_c=1)
    return panel[:, nens:].copy()


def sweep_levelwise(r, v, d, count_ops=False):
    """sherman.py:217-250 — one rank-one update per level (the paper's Step 2,
    PAPER.md:438-450).  Returns (Z, op count or None)."""
    nobs, nens = v.shape
    panel = _level0_panel(r, v, d)
    ops = 2 * nobs * nens
    for lvl in range(nens):
        vk = v[:, lvl]
        den = _checked_denominator(vk, panel[:, lvl], lvl + 1)
        h = panel[:, lvl] / den
        ops += 2 * nobs
        rest = panel[:, lvl + 1:]
        dger(-1.0, h, vk @ rest, a=rest, overwrite_a=1)
        ops += 2 * nobs * (2 * nens - lvl - 1)
    return panel[:, nens:].copy(), (ops if count_ops else None)


def solve_sherman(r, v, d, count_ops=False):
    """sherman.py:253-286 — validated solve; returns (Z, op count or None)."""
    r, v, d = validate_system(r, v, d)
    if count_ops:
        return sweep_levelwise(r, v, d, count_ops=True)
    return sweep_grouped(r, v, d), None


def analysis_step(x, perturbed, indices, r):
    """enkf.py:167-192 (unlocalized, solver="sherman", workers=1).

    X^A = X + S (V' Z) with S = member_deviations(X), V = H S,
    D = Y - H X and Z from the grouped sweep.  Returns a new array.
    """
    x = np.asarray(x, dtype=float)
    if x.ndim != 2 or x.shape[1] < 2:
        raise ValueError("analysis needs at least 2 ensemble members")
    s = member_deviations(x)
    v = apply_selection(indices, s)
    d = innovations(perturbed, indices, x)
    z, _ = solve_sherman(r, v, d)
    return x + s @ (v.T @ z)


def analysis_step_chunked(x, perturbed, indices, r, rows_per_chunk=1 << 18):
    """Row-chunked restatement of enkf.py:187-192 for inputs whose full-size
    temporaries would not fit in host RAM.  The observation
    side (V, D, Z) is formed once; the state side S and X^A are row-local,
    so chunking changes only the summation blocking of `s @ A`."""
    x = np.asarray(x, dtype=float)
    if x.ndim != 2 or x.shape[1] < 2:
        raise ValueError("analysis needs at least 2 ensemble members")
    xo = apply_selection(indices, x)
    v = member_deviations(xo)
    d = perturbed - xo
    z, _ = solve_sherman(r, v, d)
    a = v.T @ z
    out = np.empty_like(x)
    for lo in range(0, x.shape[0], rows_per_chunk):
        blk = x[lo:lo + rows_per_chunk]
        out[lo:lo + rows_per_chunk] = blk + member_deviations(blk) @ a
    return out


def influence_matrix_cyclic(nstate, indices, scale=None):
    """enkf.py:138-164: exp(-d(i, p_j) / scale), cyclic index distance;
    ``indices`` None means the identity operator (p_j = j)."""
    if scale is None:
        scale = float(nstate)
    if scale <= 0:
        raise ValueError("influence scale must be positive")
    obs_idx = np.arange(nstate) if indices is None else np.asarray(indices)
    if indices is not None and obs_idx[-1] >= nstate:
        raise ValueError("observation index out of range")
    i = np.arange(nstate)[:, None]
    raw = np.abs(i - obs_idx[None, :])
    dist = np.minimum(raw, nstate - raw)
    return np.exp(-dist / scale)


def analysis_step_localized(x, perturbed, indices, r, delta):
    """enkf.py:187-199 (localized branch): X + (Delta o (S V')) Z."""
    x = np.asarray(x, dtype=float)
    if x.ndim != 2 or x.shape[1] < 2:
        raise ValueError("analysis needs at least 2 ensemble members")
    s = member_deviations(x)
    v = apply_selection(indices, s)
    d = innovations(perturbed, indices, x)
    z, _ = solve_sherman(r, v, d)
    delta = np.asarray(delta, dtype=float)
    if delta.shape != (x.shape[0], v.shape[0]):
        raise ValueError(f"influence matrix shape {delta.shape} does not match "
                         f"(nstate, nobs) = ({x.shape[0]}, {v.shape[0]})")
    return x + (delta * (s @ v.T)) @ z


class OracleDivergence(ArithmeticError):
    """models/lorenz96.py:52-58: the state became non-finite; ``member`` is the
    first non-finite ensemble column."""

    def __init__(self, member):
        self.member = member
        super().__init__(f"state became non-finite (ensemble member {member})")


def l96_tendency(x, forcing):
    """models/lorenz96.py:31-39 (cyclic in the first axis)."""
    return (np.roll(x, -1, axis=0) - np.roll(x, 2, axis=0)) * np.roll(x, 1, axis=0) - x + forcing


def l96_rk4_step(x, dt, forcing):
    """models/lorenz96.py:42-49."""
    k1 = l96_tendency(x, forcing)
    k2 = l96_tendency(x + 0.5 * dt * k1, forcing)
    k3 = l96_tendency(x + 0.5 * dt * k2, forcing)
    k4 = l96_tendency(x + dt * k3, forcing)
    return x + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def l96_advance(x, nsteps, dt=0.05, forcing=8.0):
    """models/lorenz96.py:52-78: nsteps RK4 steps, finiteness checked after each."""
    x = np.asarray(x, dtype=float)
    for _ in range(nsteps):
        x = l96_rk4_step(x, dt, forcing)
        if not np.all(np.isfinite(x)):
            if x.ndim == 2:
                raise OracleDivergence(int(np.argmax(~np.isfinite(x).all(axis=0))))
            raise OracleDivergence(None)
    return x


def inflate(x, alpha):
    """enkf.py:123-135."""
    if alpha < 1.0:
        raise ValueError(f"inflation factor must be >= 1, got {alpha}")
    x = np.asarray(x, dtype=float)
    if alpha == 1.0:
        return x
    mean = x.mean(axis=1, keepdims=True)
    return mean + alpha * (x - mean)


def cycle_l96(x0, ys, indices, r, steps_per_cycle, dt=0.05, forcing=8.0, inflation=1.0,
              localization_scale=None):
    """experiment.py:457-479 closed loop with the lorenz96 model: forecast
    (enkf.py:202-212), inflation when > 1 (:466-467), then analysis_step — with
    the cyclic influence matrix of enkf.py:138-164 when ``localization_scale`` is
    given (experiment.py:470-473, the lorenz-small preset) — per cycle; returns the
    final ensemble and the forecast / analysis ensemble means."""
    x = np.asarray(x0, dtype=float)
    delta = None if localization_scale is None else influence_matrix_cyclic(x.shape[0], indices, localization_scale)
    mean_f, mean_a = [], []
    for y in ys:
        x = l96_advance(x, steps_per_cycle, dt, forcing)
        mean_f.append(x.mean(axis=1))
        if inflation > 1.0:
            x = inflate(x, inflation)
        x = analysis_step(x, y, indices, r) if delta is None else analysis_step_localized(x, y, indices, r, delta)
        mean_a.append(x.mean(axis=1))
    return x, np.stack(mean_f), np.stack(mean_a)
