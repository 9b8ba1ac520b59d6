"""Filter-core drop-in: `analysis_step` and its data types on the B200 path.

Mirrors `enkfkit.enkf` (reference enkf.py) for the names on the hot path:
`SelectionOperator`, `ObservationBatch`, `member_deviations`, `innovations`,
`analysis_step`.  Same signatures, argument meaning, array layout (Nstate x
Nens, C order) and error behaviour; the arithmetic runs in libenkf_b200.so
(sm_100a) and nothing falls back to the CPU.

Array types: numpy (or array-like) inputs take the host path — one C-ABI call
that copies in, runs the step and copies out — and return numpy arrays.
`torch.Tensor` inputs on a CUDA device stay device-resident and return a
CUDA tensor.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .solvers import SolverChoice, _require_sherman

try:  # torch is the device-memory / stream plumbing
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def _is_cuda_tensor(a) -> bool:
    return torch is not None and isinstance(a, torch.Tensor) and a.is_cuda


def _cuda_ready(device_index: int | None = None) -> int:
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("the EnKF analysis path needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    if device_index is None:
        device_index = torch.cuda.current_device()
    return int(device_index)


@dataclass(frozen=True)
class SelectionOperator:
    """Observation operator selecting state rows by index (enkf.py:22-59).

    ``indices`` strictly increasing and non-negative (validated at
    construction), or ``None`` for the identity.  A device copy of the index
    array is cached per CUDA device on first use.
    """

    indices: np.ndarray | None
    _device_cache: dict = field(default_factory=dict, compare=False, repr=False)

    @classmethod
    def identity(cls) -> "SelectionOperator":
        return cls(indices=None)

    @classmethod
    def from_indices(cls, indices) -> "SelectionOperator":
        if _is_cuda_tensor(indices):
            indices = indices.cpu().numpy()
        idx = np.asarray(indices, dtype=np.intp)
        if idx.ndim != 1 or idx.size < 1:
            raise ValueError("need a non-empty 1-D index array")
        if np.any(np.diff(idx) <= 0):
            raise ValueError("indices must be strictly increasing")
        if idx[0] < 0:
            raise ValueError("indices must be non-negative")
        return cls(indices=np.ascontiguousarray(idx, dtype=np.int64))

    def nobs(self, nstate: int) -> int:
        return nstate if self.indices is None else int(self.indices.size)

    def check_range(self, nstate: int) -> None:
        """The IndexError of enkf.py:54-58."""
        if self.indices is not None and self.indices[-1] >= nstate:
            raise IndexError(f"observation index {self.indices[-1]} out of range "
                             f"for state size {nstate}")

    def device_indices(self, device):
        if self.indices is None:
            return None
        key = str(device)
        t = self._device_cache.get(key)
        if t is None:
            t = torch.from_numpy(np.ascontiguousarray(self.indices, dtype=np.int64)).to(device)
            self._device_cache[key] = t
        return t

    def apply(self, x):
        """Select observed rows (identity returns ``x`` itself, enkf.py:50-59)."""
        if self.indices is None:
            return x
        self.check_range(x.shape[0])
        if _is_cuda_tensor(x):
            return x.index_select(0, self.device_indices(x.device))
        return x[self.indices]


@dataclass(frozen=True)
class ObservationBatch:
    """One observation vector and its per-member perturbed copies
    (enkf.py:62-71): ``perturbed[:, j] == y + perturbations[:, j]``."""

    y: object
    perturbed: object
    perturbations: object


def _f64_contig_device(a, device):
    if _is_cuda_tensor(a):
        t = a
        if t.device != device:
            t = t.to(device)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(device)
    if t.dtype != torch.float64:
        t = t.to(torch.float64)
    return t.contiguous()


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def member_deviations(x):
    """S = (X - row mean) / sqrt(N - 1) on the GPU (enkf.py:82-92)."""
    dev_in = _is_cuda_tensor(x)
    if not dev_in:
        x = np.asarray(x, dtype=float)
    if x.ndim != 2 or x.shape[1] < 2:
        raise ValueError("need at least 2 ensemble members for deviations")
    device = torch.device("cuda", _cuda_ready(x.device.index if dev_in else None))
    xd = _f64_contig_device(x, device)
    out = torch.empty_like(xd)
    with _native.on_device(device.index):
        code = _native.lib().enkf_member_deviations_f64(
            xd.data_ptr(), out.data_ptr(), xd.shape[0], xd.shape[1], _stream_ptr(device))
    _native.raise_for_status(code, None, "enkf_member_deviations_f64")
    return out if dev_in else out.cpu().numpy()


def inflate(x, alpha: float):
    """Scale deviations about the ensemble mean by alpha >= 1 on the GPU
    (enkf.py:123-135; alpha == 1 returns the input as a float array)."""
    if alpha < 1.0:
        raise ValueError(f"inflation factor must be >= 1, got {alpha}")
    dev_in = _is_cuda_tensor(x)
    if not dev_in:
        x = np.asarray(x, dtype=float)
    if alpha == 1.0:
        return x
    if x.ndim != 2:
        raise ValueError("inflate expects an (nstate, nens) ensemble")
    device = torch.device("cuda", _cuda_ready(x.device.index if dev_in else None))
    xd = _f64_contig_device(x, device)
    out = torch.empty_like(xd)
    with _native.on_device(device.index):
        code = _native.lib().enkf_inflate_f64(xd.data_ptr(), out.data_ptr(), xd.shape[0], xd.shape[1],
                                              float(alpha), _stream_ptr(device))
    _native.raise_for_status(code, None, "enkf_inflate_f64")
    return out if dev_in else out.cpu().numpy()


def innovations(obs: ObservationBatch, h: SelectionOperator, x):
    """D = Y - H(X) on the GPU (enkf.py:114-120)."""
    dev_in = _is_cuda_tensor(x)
    if not dev_in:
        x = np.asarray(x, dtype=float)
    h.check_range(x.shape[0])
    device = torch.device("cuda", _cuda_ready(x.device.index if dev_in else None))
    xd = _f64_contig_device(x, device)
    yd = _f64_contig_device(obs.perturbed, device)
    nobs = h.nobs(xd.shape[0])
    if yd.dim() != 2 or yd.shape[0] != nobs or (xd.dim() == 2 and yd.shape[1] != xd.shape[1]):
        raise ValueError(f"perturbed observations {tuple(yd.shape)} do not match "
                         f"H(x) ({nobs}, {xd.shape[1] if xd.dim() == 2 else 1})")
    out = torch.empty_like(yd)
    idx = h.device_indices(device)
    with _native.on_device(device.index):
        code = _native.lib().enkf_innovations_f64(
            xd.data_ptr(), yd.data_ptr(), 0 if idx is None else idx.data_ptr(),
            out.data_ptr(), nobs, yd.shape[1], _stream_ptr(device))
    _native.raise_for_status(code, None, "enkf_innovations_f64")
    return out if dev_in else out.cpu().numpy()


_PINNED_RESULT_BYTES = 64 << 20


def _host_result(shape) -> np.ndarray:
    """A new C-order float64 result array.  Large results live in page-locked
    memory from torch's caching host allocator, so the device->host copy runs at
    full PCIe speed straight into the caller's array (fresh pageable pages
    fault at a few GB/s); the block returns to the cache when the array dies."""
    nbytes = int(np.prod(shape)) * 8
    if nbytes >= _PINNED_RESULT_BYTES:
        return torch.empty(tuple(shape), dtype=torch.float64, pin_memory=True).numpy()
    return np.empty(shape, dtype=np.float64)


def _check_obs_shapes(nobs: int, nens: int, perturbed_shape, r_shape):
    if nobs == 0:
        # the reference fails on an empty observation set too: ValueError from the
        # first rank-1 update of its empty panel (sherman.py:187)
        raise ValueError("the Sherman-Morrison sweep needs at least one observation")
    if len(perturbed_shape) != 2 or tuple(perturbed_shape) != (nobs, nens):
        raise ValueError(f"perturbed observations have shape {tuple(perturbed_shape)}, "
                         f"expected ({nobs}, {nens})")
    if len(r_shape) != 1:
        raise ValueError(f"r must be a vector, got shape {tuple(r_shape)}")
    if r_shape[0] != nobs:
        raise ValueError(f"row mismatch: r has {r_shape[0]}, V has {nobs}, D has {nobs}")


def analysis_step(
    x,
    obs: ObservationBatch,
    h: SelectionOperator,
    r,
    solver: SolverChoice | str = SolverChoice.SHERMAN,
    localization=None,
    workers: int = 1,
):
    """One stochastic-EnKF analysis update, X^A = X + S (V'Z) (enkf.py:167-192).

    Same signature as the reference.  ``solver`` must be "sherman" (the other
    reference solvers are not on this path); ``workers`` is accepted and
    ignored (the GPU result does not depend on it).  ``localization`` is the
    (nstate, nobs) influence matrix of enkf.py:193-199: a dense array/tensor,
    or the lazy ``influence_matrix_cyclic`` object, which is evaluated on the
    fly (matrix-free).  Returns a new array; inputs are never modified.
    """
    _require_sherman(solver)
    dev_in = _is_cuda_tensor(x)
    if not dev_in:
        x = np.asarray(x, dtype=float)
    if x.ndim != 2 or x.shape[1] < 2:
        raise ValueError("analysis needs at least 2 ensemble members")
    nstate, nens = int(x.shape[0]), int(x.shape[1])
    if nens > _native.max_ens():
        raise NotImplementedError(f"n_ens={nens} exceeds the supported maximum {_native.max_ens()}")
    h.check_range(nstate)
    nobs = h.nobs(nstate)
    perturbed = obs.perturbed
    if not _is_cuda_tensor(perturbed):
        perturbed = np.asarray(perturbed, dtype=float)
    if _is_cuda_tensor(r):
        # device-resident r: its positivity / finiteness is checked by the Gram pass
        # (FLAG_R_NONPOS / FLAG_NONFINITE -> the same ValueError), without a host copy
        r_host = None
        _check_obs_shapes(nobs, nens, tuple(perturbed.shape), tuple(r.shape))
    else:
        r_host = np.asarray(r, dtype=float)
        _check_obs_shapes(nobs, nens, tuple(perturbed.shape), r_host.shape)
        if np.any(r_host <= 0):
            raise ValueError("observation variances must be positive")
        if not np.all(np.isfinite(r_host)):
            raise ValueError("inputs contain non-finite entries")

    if localization is not None:
        return _analysis_localized(x, perturbed, h, r, localization, nstate, nobs, nens, dev_in)

    if dev_in:
        device = x.device
        _cuda_ready(device.index)
        plan = _native.get_plan(device.index, nstate, nobs, nens)
        xd = _f64_contig_device(x, device)
        yd = _f64_contig_device(perturbed, device)
        rd = _f64_contig_device(r, device)
        idx = h.device_indices(device)
        out = torch.empty_like(xd)
        st = _native.EnkfStatus()
        with plan.lock:
            code = _native.lib().enkf_analysis_f64(
                plan.handle, xd.data_ptr(), yd.data_ptr(),
                0 if idx is None else idx.data_ptr(), rd.data_ptr(), out.data_ptr(),
                _stream_ptr(device), ctypes.byref(st))
        _native.raise_for_status(code, st, "enkf_analysis_f64")
        return out

    device_index = _cuda_ready()
    plan = _native.get_plan(device_index, nstate, nobs, nens)
    if r_host is None:  # host x with a device-resident r
        r_host = r.detach().cpu().numpy()
    xh = np.ascontiguousarray(x, dtype=np.float64)
    yh = np.ascontiguousarray(perturbed, dtype=np.float64)
    rh = np.ascontiguousarray(r_host, dtype=np.float64)
    idxh = None if h.indices is None else np.ascontiguousarray(h.indices, dtype=np.int64)
    out = _host_result(xh.shape)
    st = _native.EnkfStatus()
    with plan.lock:
        code = _native.lib().enkf_analysis_host_f64(
            plan.handle, xh.ctypes.data, yh.ctypes.data,
            None if idxh is None else idxh.ctypes.data, rh.ctypes.data, out.ctypes.data,
            ctypes.byref(st))
    _native.raise_for_status(code, st, "enkf_analysis_host_f64")
    return out


class CyclicInfluence:
    """Lazy ``influence_matrix_cyclic`` (enkf.py:138-164).

    Entry (i, j) is exp(-d(i, p_j) / scale), d the cyclic index distance
    min(|i - p|, nstate - |i - p|) and p_j the state index of observation j.
    ``np.asarray(obj)`` materialises exactly the reference's dense matrix (and
    indexing / ``min`` / ``max`` go through it), but ``analysis_step`` never
    does: it evaluates the taper inside the localized-update kernel, so the
    Nstate x Nobs matrix is not formed at any size.
    """

    ndim = 2
    dtype = np.dtype(np.float64)

    def __init__(self, nstate: int, h: SelectionOperator, scale: float):
        self.nstate = int(nstate)
        self.h = h
        self.scale = float(scale)
        self.shape = (self.nstate, h.nobs(self.nstate))

    def _obs_idx(self):
        return np.arange(self.nstate) if self.h.indices is None else self.h.indices

    def __array__(self, dtype=None, copy=None):
        i = np.arange(self.nstate)[:, None]
        raw = np.abs(i - self._obs_idx()[None, :])
        dist = np.minimum(raw, self.nstate - raw)
        out = np.exp(-dist / self.scale)
        return out if dtype is None else out.astype(dtype)

    def __getitem__(self, key):
        return np.asarray(self)[key]

    def min(self):
        return np.asarray(self).min()

    def max(self):
        return np.asarray(self).max()

    def same_operator(self, h: SelectionOperator) -> bool:
        if self.h.indices is None or h.indices is None:
            return self.h.indices is None and h.indices is None
        return self.h.indices.shape == h.indices.shape and bool(np.array_equal(self.h.indices, h.indices))


def influence_matrix_cyclic(nstate: int, h: SelectionOperator, scale: float | None = None) -> CyclicInfluence:
    """Distance-based impact factors for a periodic 1-D state (enkf.py:138-164):
    same arguments, defaults and ValueErrors as the reference; returns the lazy
    :class:`CyclicInfluence` (array-convertible to the reference's matrix)."""
    if scale is None:
        scale = float(nstate)
    if scale <= 0:
        raise ValueError("influence scale must be positive")
    if h.indices is not None and h.indices[-1] >= nstate:
        raise ValueError("observation index out of range")
    return CyclicInfluence(nstate, h, scale)


def _analysis_localized(x, perturbed, h, r, localization, nstate, nobs, nens, dev_in):
    """enkf.py:193-199: X + (Delta o (S V')) Z on the GPU (localized_update_kernel)."""
    cyclic = isinstance(localization, CyclicInfluence) and localization.same_operator(h) \
        and localization.nstate == nstate
    if cyclic:
        shape = localization.shape
    elif _is_cuda_tensor(localization):
        shape = tuple(localization.shape)
    else:
        localization = np.asarray(localization, dtype=float)
        shape = localization.shape
    if tuple(shape) != (nstate, nobs):
        raise ValueError(f"influence matrix shape {tuple(shape)} does not match "
                         f"(nstate, nobs) = ({nstate}, {nobs})")
    device = torch.device("cuda", _cuda_ready(x.device.index if dev_in else None))
    plan = _native.get_plan(device.index, nstate, nobs, nens)
    xd = _f64_contig_device(x, device)
    yd = _f64_contig_device(perturbed, device)
    rd = _f64_contig_device(r, device)
    idx = h.device_indices(device)
    out = torch.empty_like(xd)
    st = _native.EnkfStatus()
    with plan.lock:
        if cyclic:
            code = _native.lib().enkf_analysis_localized_cyclic_f64(
                plan.handle, xd.data_ptr(), yd.data_ptr(), 0 if idx is None else idx.data_ptr(),
                rd.data_ptr(), localization.scale, out.data_ptr(), _stream_ptr(device), ctypes.byref(st))
        else:
            dd = _f64_contig_device(localization, device)
            code = _native.lib().enkf_analysis_localized_f64(
                plan.handle, xd.data_ptr(), yd.data_ptr(), 0 if idx is None else idx.data_ptr(),
                rd.data_ptr(), dd.data_ptr(), out.data_ptr(), _stream_ptr(device), ctypes.byref(st))
    _native.raise_for_status(code, st, "enkf_analysis_localized_f64")
    return out if dev_in else out.cpu().numpy()
