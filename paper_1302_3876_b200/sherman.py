"""Iterative Sherman-Morrison solve on the GPU (drop-in for reference sherman.py).

Solves (diag(r) + V V') Z = D.  The reference sweeps one rank-one update per
ensemble column over the Nobs x 2N workspace G = [V/r | D/r] (sherman.py:1-36,
157-214), streaming the workspace once per group of GROUP_LEVELS levels.  On
B200 the same rank-one sequence is applied in reduced coordinates: one HBM
pass forms the level-0 Gram [V'R^-1 V | V'R^-1 D] (the dot products every
level needs), the N levels run on that N x 2N Gram in one SM's shared memory
(den_k = 1 + v_k'u_k, the 1e-14 guard, the composition), and a second pass
writes Z = R^-1 (D - V A) with A = V'Z.  All N levels are fused per HBM pass,
the limit of the reference's group width.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _native

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

# sherman.py:51 / :146 (GROUP_LEVELS is the reference's CPU blocking width; the
# GPU path fuses all levels and exports the constant for API parity only).
SINGULAR_TOL = 1e-14
GROUP_LEVELS = 8


@dataclass
class SolverResult:
    """sherman.py:54-70."""

    z: object
    seconds: float
    long_ops: int | None = None


def long_op_count(nens: int, nobs: int) -> int:
    """sherman.py:73-82 — 3 (N^2 Nobs + N Nobs) multiplications and divisions."""
    if nens < 1 or nobs < 1:
        raise ValueError("nens and nobs must be at least 1")
    return 3 * (nens * nens * nobs + nens * nobs)


def _partition(lo: int, hi: int, parts: int):
    """sherman.py:111-125 — contiguous blocks differing in size by at most one."""
    span = hi - lo
    parts = min(parts, span)
    if parts <= 0:
        return []
    size, extra = divmod(span, parts)
    out, start = [], lo
    for i in range(parts):
        stop = start + size + (i < extra)
        out.append((start, stop))
        start = stop
    return out


def level_blocks(nens: int, level: int, workers: int):
    """sherman.py:128-139 — column blocks a level's update is split into."""
    if not 0 <= level <= nens:
        raise ValueError(f"level must be in [0, {nens}], got {level}")
    if workers < 1:
        raise ValueError("workers must be at least 1")
    return _partition(level, 2 * nens, workers)


def _is_cuda_tensor(a) -> bool:
    return torch is not None and isinstance(a, torch.Tensor) and a.is_cuda


def _validate_host(r, v, d):
    """sherman.py:85-108 (numpy inputs are validated on the host before any
    device work, so the error precedence matches the reference)."""
    r = np.asarray(r, dtype=float)
    v = np.asarray(v, dtype=float)
    d = np.asarray(d, dtype=float)
    if r.ndim != 1:
        raise ValueError(f"r must be a vector, got shape {r.shape}")
    if v.ndim != 2 or d.ndim != 2:
        raise ValueError("V and D must be matrices")
    if v.shape[0] != r.shape[0] or d.shape[0] != r.shape[0]:
        raise ValueError(f"row mismatch: r has {r.shape[0]}, V has {v.shape[0]}, D has {d.shape[0]}")
    if v.shape[1] != d.shape[1]:
        raise ValueError(f"column mismatch: V has {v.shape[1]}, D has {d.shape[1]}")
    if v.shape[1] < 1:
        raise ValueError("need at least one ensemble column")
    if v.shape[0] < 1:  # the reference's sweep raises ValueError on an empty panel (sherman.py:187)
        raise ValueError("the Sherman-Morrison sweep needs at least one observation")
    if np.any(r <= 0):
        raise ValueError("observation variances must be positive")
    if not (np.all(np.isfinite(v)) and np.all(np.isfinite(d)) and np.all(np.isfinite(r))):
        raise ValueError("inputs contain non-finite entries")
    return r, v, d


def _validate_shapes_device(r, v, d):
    if r.dim() != 1:
        raise ValueError(f"r must be a vector, got shape {tuple(r.shape)}")
    if v.dim() != 2 or d.dim() != 2:
        raise ValueError("V and D must be matrices")
    if v.shape[0] != r.shape[0] or d.shape[0] != r.shape[0]:
        raise ValueError("row mismatch between r, V and D")
    if v.shape[1] != d.shape[1]:
        raise ValueError("column mismatch between V and D")
    if v.shape[1] < 1:
        raise ValueError("need at least one ensemble column")
    if v.shape[0] < 1:  # the reference's sweep raises ValueError on an empty panel (sherman.py:187)
        raise ValueError("the Sherman-Morrison sweep needs at least one observation")


def _solve_device(r, v, d, return_a: bool = False):
    """Run enkf_ism_solve_f64 on CUDA tensors; returns (Z, A)."""
    device = v.device
    nobs, nens = int(v.shape[0]), int(v.shape[1])
    if nens > _native.max_ens():
        raise NotImplementedError(f"n_ens={nens} exceeds the supported maximum {_native.max_ens()}")
    plan = _native.get_plan(device.index, 0, nobs, nens)
    rd = r.to(device=device, dtype=torch.float64).contiguous()
    vd = v.to(torch.float64).contiguous()
    dd = d.to(device=device, dtype=torch.float64).contiguous()
    z = torch.empty_like(dd)
    a = torch.empty((nens, nens), dtype=torch.float64, device=device)
    st = _native.EnkfStatus()
    with plan.lock:
        code = _native.lib().enkf_ism_solve_f64(
            plan.handle, rd.data_ptr(), vd.data_ptr(), dd.data_ptr(), z.data_ptr(),
            a.data_ptr(), torch.cuda.current_stream(device).cuda_stream, ctypes.byref(st))
    _native.raise_for_status(code, st, "enkf_ism_solve_f64")
    return z, a


def solve_sherman(r, v, d, *, count_ops: bool = False, verify_frozen: bool = False) -> SolverResult:
    """sherman.py:253-286 — solve (diag(r) + V V') Z = D on the GPU.

    ``count_ops`` reports the closed-form long-operation count (the reference's
    instrumented counter equals it exactly, tests/test_sherman.py:165-179).
    ``verify_frozen`` is accepted: finished pivot columns are never stored on
    the GPU path, so the reference's frozen-column assertion holds trivially.
    """
    del verify_frozen
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("solve_sherman needs a CUDA device (no CPU fallback)")
    if _is_cuda_tensor(v):
        rt = r if _is_cuda_tensor(r) else torch.as_tensor(np.asarray(r, dtype=float), device=v.device)
        dt = d if _is_cuda_tensor(d) else torch.as_tensor(np.asarray(d, dtype=float), device=v.device)
        _validate_shapes_device(rt, v, dt)
        t0 = time.perf_counter()
        z, _ = _solve_device(rt, v, dt)
        torch.cuda.synchronize(v.device)
        seconds = time.perf_counter() - t0
        nobs, nens = int(v.shape[0]), int(v.shape[1])
    else:
        r, v, d = _validate_host(r, v, d)
        nobs, nens = v.shape
        dev = torch.device("cuda", torch.cuda.current_device())
        t0 = time.perf_counter()
        zt, _ = _solve_device(torch.from_numpy(r).to(dev), torch.from_numpy(np.ascontiguousarray(v)).to(dev),
                              torch.from_numpy(np.ascontiguousarray(d)).to(dev))
        z = zt.cpu().numpy()
        seconds = time.perf_counter() - t0
    ops = long_op_count(nens, nobs) if count_ops else None
    return SolverResult(z=z, seconds=seconds, long_ops=ops)


def solve_sherman_blocked(r, v, d, workers: int = 1) -> SolverResult:
    """sherman.py:289-311 — the thread-blocked variant.  The GPU sweep has a
    fixed reduction order, so every ``workers`` value gives the bitwise-same
    result as `solve_sherman`."""
    if workers < 1:
        raise ValueError("workers must be at least 1")
    return solve_sherman(r, v, d)
