"""Device-resident Lorenz-96 forecasts and the cycled driver.

Mirrors the reference's model operator (models/lorenz96.py:18-89) and
`forecast_step` (enkf.py:202-212); the arithmetic runs in libenkf_b200.so
(`enkf_forecast_l96_f64`, bit-identical to the reference's numpy RK4).
`cycle_l96` runs the experiment.py:457-479 loop (forecast -> analysis for every
cycle) on the GPU without host round trips between cycles, with the perturbed
observations of all cycles pre-staged on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .enkf import SelectionOperator, _cuda_ready, _f64_contig_device, _is_cuda_tensor, _stream_ptr
from .errors import NumericalFailureError

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


@dataclass(frozen=True)
class Lorenz96Config:
    """lorenz96.py:18-28."""

    nstate: int
    forcing: float = 8.0
    dt: float = 0.05

    def __post_init__(self):
        if self.nstate < 4:
            raise ValueError("the periodic stencil needs at least 4 variables")
        if self.dt <= 0:
            raise ValueError("dt must be positive")


def _window_steps(t0: float, t1: float, dt: float) -> int:
    """lorenz96.py:80-89."""
    if t1 < t0:
        raise ValueError(f"window is reversed: {t0} > {t1}")
    nsteps = round((t1 - t0) / dt)
    if abs(nsteps * dt - (t1 - t0)) > 1e-9 * max(1.0, abs(t1 - t0)):
        raise ValueError(f"window [{t0}, {t1}] is not a whole number of steps of dt={dt}")
    return nsteps


def _run(x, nsteps: int, cfg: Lorenz96Config):
    dev_in = _is_cuda_tensor(x)
    if not dev_in:
        x = np.asarray(x, dtype=float)
    if x.shape[0] < 4:
        raise ValueError("state must have at least 4 components")
    one_d = x.ndim == 1
    device = torch.device("cuda", _cuda_ready(x.device.index if dev_in else None))
    xd = _f64_contig_device(x, device)
    if one_d:
        xd = xd.reshape(-1, 1)
    ns, nens = int(xd.shape[0]), int(xd.shape[1])
    plan = _native.get_plan(device.index, ns, 1, nens)
    out = torch.empty_like(xd)
    st = _native.EnkfStatus()
    with plan.lock:
        code = _native.lib().enkf_forecast_l96_f64(plan.handle, xd.data_ptr(), out.data_ptr(), cfg.dt,
                                                   cfg.forcing, int(nsteps), _stream_ptr(device), ctypes.byref(st))
    _native.raise_for_status(code, st, "enkf_forecast_l96_f64")
    if one_d:
        out = out.reshape(-1)
    return out if dev_in else out.cpu().numpy()


class Lorenz96:
    """Model operator advancing states with fixed-step RK4 (lorenz96.py:61-78),
    on the GPU.  Accepts a single state (n,) or an ensemble (n, m), numpy or
    CUDA tensor; a non-finite state raises DivergenceError(member)."""

    def __init__(self, config: Lorenz96Config):
        self.config = config

    def step(self, x):
        return _run(x, 1, self.config)

    def advance(self, x, t0: float, t1: float):
        return _run(x, _window_steps(t0, t1, self.config.dt), self.config)


def forecast_step(model, x, t0: float, t1: float):
    """enkf.py:202-212: advance every ensemble column with the model operator."""
    if t1 < t0:
        raise ValueError(f"forecast window is reversed: {t0} > {t1}")
    if t1 == t0:
        return x if _is_cuda_tensor(x) else np.asarray(x, dtype=float)
    return model.advance(x if _is_cuda_tensor(x) else np.asarray(x, dtype=float), t0, t1)


@dataclass
class CycleResult:
    """Final analysis ensemble and the per-cycle forecast / analysis ensemble
    means (the quantities the reference's cycle_error reads, experiment.py:426-430)."""

    x: object        # (nstate, nens) CUDA tensor
    mean_f: object   # (cycles, nstate) CUDA tensor
    mean_a: object   # (cycles, nstate) CUDA tensor


def cycle_l96(model: Lorenz96, x0, perturbed, h: SelectionOperator, r, steps_per_cycle: int,
              inflation: float = 1.0, localization_scale: float | None = None) -> CycleResult:
    """Closed-loop cycling on the device: for every cycle c, X <- forecast(X,
    steps_per_cycle RK4 steps); X <- inflate(X, inflation) when inflation > 1
    (experiment.py:466-467); X <- analysis_step(X, perturbed[c], h, r), localized
    with influence_matrix_cyclic(nstate, h, localization_scale) when a scale is
    given (experiment.py:470-473; the taper is evaluated in-kernel).

    ``perturbed``: (cycles, nobs, nens) pre-staged perturbed observations
    (numpy or CUDA tensor).  Failures raise NumericalFailureError naming the
    cycle (1-based, as experiment.py:474-478) chained to the underlying
    SingularUpdateError / DivergenceError / ValueError."""
    cfg = model.config
    if inflation < 1.0:
        raise ValueError(f"inflation factor must be >= 1, got {inflation}")
    if localization_scale is not None and not localization_scale > 0:
        raise ValueError("influence scale must be positive")
    dev_in = _is_cuda_tensor(x0)
    device = torch.device("cuda", _cuda_ready(x0.device.index if dev_in else None))
    x = _f64_contig_device(x0, device).clone()
    if x.dim() != 2 or x.shape[1] < 2:
        raise ValueError("analysis needs at least 2 ensemble members")
    ns, nens = int(x.shape[0]), int(x.shape[1])
    if ns != cfg.nstate:
        raise ValueError(f"ensemble has {ns} rows, model nstate is {cfg.nstate}")
    h.check_range(ns)
    nobs = h.nobs(ns)
    ys = _f64_contig_device(perturbed, device)
    if ys.dim() != 3 or tuple(ys.shape[1:]) != (nobs, nens):
        raise ValueError(f"perturbed observations have shape {tuple(ys.shape)}, expected (cycles, {nobs}, {nens})")
    r_host = r.detach().cpu().numpy() if _is_cuda_tensor(r) else np.asarray(r, dtype=float)
    if r_host.shape != (nobs,):
        raise ValueError(f"r has shape {r_host.shape}, expected ({nobs},)")
    if np.any(r_host <= 0):
        raise ValueError("observation variances must be positive")
    cycles = int(ys.shape[0])
    rd = _f64_contig_device(r_host, device)
    idx = h.device_indices(device)
    mean_f = torch.empty((cycles, ns), dtype=torch.float64, device=device)
    mean_a = torch.empty((cycles, ns), dtype=torch.float64, device=device)
    plan = _native.get_plan(device.index, ns, nobs, nens)
    st = _native.EnkfStatus()
    failed = ctypes.c_int32(-1)
    with plan.lock:
        if localization_scale is None:
            code = _native.lib().enkf_cycle_l96_f64(
                plan.handle, x.data_ptr(), ys.data_ptr(), 0 if idx is None else idx.data_ptr(), rd.data_ptr(),
                cycles, int(steps_per_cycle), cfg.dt, cfg.forcing, float(inflation), mean_f.data_ptr(),
                mean_a.data_ptr(), _stream_ptr(device), ctypes.byref(st), ctypes.byref(failed))
        else:
            code = _native.lib().enkf_cycle_l96_localized_f64(
                plan.handle, x.data_ptr(), ys.data_ptr(), 0 if idx is None else idx.data_ptr(), rd.data_ptr(),
                cycles, int(steps_per_cycle), cfg.dt, cfg.forcing, float(inflation), float(localization_scale),
                mean_f.data_ptr(), mean_a.data_ptr(), _stream_ptr(device), ctypes.byref(st), ctypes.byref(failed))
    if code != _native.ENKF_OK:
        try:
            _native.raise_for_status(code, st, "enkf_cycle_l96_f64")
        except ArithmeticError as exc:
            raise NumericalFailureError(f"solver 'sherman' failed at cycle {failed.value + 1}: {exc}") from exc
    return CycleResult(x=x, mean_f=mean_f, mean_a=mean_a)
