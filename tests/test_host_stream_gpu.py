"""The streamed host-buffer path of enkf_analysis_host_f64 (page-locked X and
X^A): observed rows gathered over PCIe by gather_rows_kernel, the Gram pass on
the compact rows, X chunks in / X^A chunks out on two copy streams.  It must
equal the serial host path and the device-resident path bit for bit (same
kernels, same row order), at ragged chunk boundaries, and keep the index and
validation errors of the reference (enkf.py:54-58, sherman.py:85-108)."""

import ctypes
import os

import numpy as np
import pytest

import oracle
from golden_io import rel_err
import paper_1302_3876_b200 as P
from paper_1302_3876_b200 import _native
from paper_1302_3876_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1302_3876_b200.build import build
    build()
    import torch
    assert torch.cuda.is_available()


def _pinned(a):
    import torch
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def _plan(shape, monkeypatch, **env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    plan = _native.Plan(*shape, 0)
    for k in env:
        monkeypatch.delenv(k)
    return plan


def _host_call(plan, x, y, idx, r, out):
    st = _native.EnkfStatus()
    rc = _native.lib().enkf_analysis_host_f64(plan.handle, x.ctypes.data, y.ctypes.data,
                                             None if idx is None else idx.ctypes.data, r.ctypes.data,
                                             out.ctypes.data, ctypes.byref(st))
    return rc, st


@pytest.mark.parametrize("maker", ["config4s8", "config3", "config4s10"])
def test_streamed_equals_serial_and_device(maker, monkeypatch):
    import torch
    p = {"config4s8": lambda: W.config4(8), "config4s10": lambda: W.config4(10), "config3": W.config3}[maker]()
    assert p.indices is not None
    shape = (p.x.shape[0], p.perturbed.shape[0], p.x.shape[1])
    x, y = _pinned(p.x), _pinned(p.perturbed)
    idx = np.ascontiguousarray(p.indices, dtype=np.int64)
    r = np.ascontiguousarray(p.r)
    # 1024-row chunks (the minimum): many chunks, the last one ragged
    streamed = _plan(shape, monkeypatch, ENKF_HOST_CHUNK_MB="0")
    serial = _plan(shape, monkeypatch, ENKF_HOST_STREAM="0")
    out_s, out_q = _pinned(np.zeros_like(p.x)), _pinned(np.zeros_like(p.x))
    rc, st = _host_call(streamed, x, y, idx, r, out_s)
    assert rc == 0, st.message
    rc, st = _host_call(serial, x, y, idx, r, out_q)
    assert rc == 0, st.message
    assert np.array_equal(out_s, out_q)
    dev = torch.device("cuda", 0)
    obs = P.ObservationBatch(y=None, perturbed=torch.from_numpy(p.perturbed).to(dev), perturbations=None)
    xa_d = P.analysis_step(torch.from_numpy(p.x).to(dev), obs, P.SelectionOperator.from_indices(p.indices),
                           torch.from_numpy(p.r).to(dev))
    assert np.array_equal(xa_d.cpu().numpy(), out_s)
    assert rel_err(out_s, oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)) <= 1e-9
    # inputs untouched
    assert np.array_equal(x, p.x) and np.array_equal(y, p.perturbed)


def test_public_api_with_pinned_inputs_takes_streamed_path():
    p = W.config4(8)
    x, y = _pinned(p.x), _pinned(p.perturbed)
    obs = P.ObservationBatch(y=p.y, perturbed=y, perturbations=None)
    xa = P.analysis_step(x, obs, P.SelectionOperator.from_indices(p.indices), p.r)
    xa_pageable = P.analysis_step(p.x, P.ObservationBatch(y=p.y, perturbed=p.perturbed, perturbations=None),
                                  P.SelectionOperator.from_indices(p.indices), p.r)
    assert np.array_equal(xa, xa_pageable)
    assert not np.shares_memory(xa, x)


def test_streamed_path_errors(monkeypatch):
    """Index range / order and non-finite / non-positive inputs come back as the
    reference's errors from the streamed path, and the plan stays usable."""
    rng = np.random.default_rng(5)
    ns, nobs, n = 6000, 700, 128
    x = _pinned(rng.standard_normal((ns, n)))
    y = _pinned(rng.standard_normal((nobs, n)))
    r = np.ones(nobs)
    good = np.sort(rng.choice(ns, nobs, replace=False)).astype(np.int64)
    plan = _plan((ns, nobs, n), monkeypatch, ENKF_HOST_CHUNK_MB="0")
    out = _pinned(np.zeros((ns, n)))
    bad_range = good.copy()
    bad_range[-1] = ns + 10**9  # would be far outside the pinned block: must not be read
    bad_order = good.copy()
    bad_order[5] = bad_order[4]
    for idx, code in ((bad_range, _native.ENKF_INDEX_RANGE), (bad_order, _native.ENKF_INVALID_ARGUMENT)):
        rc, st = _host_call(plan, x, y, idx, r, out)
        assert rc == code, st.message
    r_bad = r.copy()
    r_bad[3] = -1.0
    rc, st = _host_call(plan, x, y, good, r_bad, out)
    assert rc == _native.ENKF_INVALID_ARGUMENT and b"positive" in st.message
    x_nan = x.copy()
    x_nan[good[17], 3] = np.nan
    x_nan = _pinned(x_nan)
    rc, st = _host_call(plan, x_nan, y, good, r, out)
    assert rc == _native.ENKF_INVALID_ARGUMENT and b"non-finite" in st.message
    # an unobserved non-finite row is not an error (the reference only validates V, D)
    unobs = np.setdiff1d(np.arange(ns), good)[0]
    x_u = x.copy()
    x_u[unobs, 0] = np.inf
    x_u = _pinned(x_u)
    rc, st = _host_call(plan, x_u, y, good, r, out)
    assert rc == 0, st.message
    assert not np.all(np.isfinite(out[unobs]))
    rc, st = _host_call(plan, x, y, good, r, out)
    assert rc == 0, st.message
    assert rel_err(out, oracle.analysis_step(np.array(x), np.array(y), good, r)) <= 1e-9


@pytest.mark.parametrize("xa_pinned", [False, True])
def test_pageable_streamed_equals_device(xa_pinned, monkeypatch):
    """The pageable form of the streamed host path (the caller's ordinary arrays:
    observed rows gathered on the host, X in and X^A out through pinned rings while
    the anomaly update runs chunk by chunk): 1 MiB ring slots give 1024-row chunks,
    the last one ragged; bit-equal to the device-resident step, with a pageable or a
    page-locked X^A."""
    import torch
    p = W.config4(8)
    x = np.array(p.x[:-333])  # 65203 rows: 63 full 1024-row chunks and a ragged one
    idx = np.ascontiguousarray(p.indices, dtype=np.int64)
    keep = idx < x.shape[0]
    idx, y, r = idx[keep], np.ascontiguousarray(p.perturbed[keep]), np.ascontiguousarray(p.r[keep])
    out = _pinned(np.zeros_like(x)) if xa_pinned else np.zeros_like(x)
    plan = _plan((x.shape[0], idx.size, x.shape[1]), monkeypatch, ENKF_HOST_STREAM_MIN_MB="0", ENKF_HOST_RING_MB="1")
    rc, st = _host_call(plan, x, y, idx, r, out)
    assert rc == 0, st.message
    dev = torch.device("cuda", 0)
    obs = P.ObservationBatch(y=None, perturbed=torch.from_numpy(y).to(dev), perturbations=None)
    xa_d = P.analysis_step(torch.from_numpy(x).to(dev), obs, P.SelectionOperator.from_indices(idx),
                           torch.from_numpy(r).to(dev))
    assert np.array_equal(xa_d.cpu().numpy(), out)
    assert rel_err(out, oracle.analysis_step(x, y, idx, r)) <= 1e-9


def test_pageable_streamed_errors(monkeypatch):
    """Index range / order (checked on the host before the gather) and non-finite /
    non-positive inputs (device flags) through the pageable streamed path."""
    rng = np.random.default_rng(7)
    ns, nobs, n = 6000, 700, 128
    x = rng.standard_normal((ns, n))
    y = rng.standard_normal((nobs, n))
    r = np.ones(nobs)
    good = np.sort(rng.choice(ns, nobs, replace=False)).astype(np.int64)
    plan = _plan((ns, nobs, n), monkeypatch, ENKF_HOST_STREAM_MIN_MB="0", ENKF_HOST_RING_MB="1")
    out = np.zeros((ns, n))
    bad_range = good.copy()
    bad_range[-1] = ns + 10**9  # must not be read
    bad_order = good.copy()
    bad_order[5] = bad_order[4]
    for idx, code in ((bad_range, _native.ENKF_INDEX_RANGE), (bad_order, _native.ENKF_INVALID_ARGUMENT)):
        rc, st = _host_call(plan, x, y, idx, r, out)
        assert rc == code, st.message
    r_bad = r.copy()
    r_bad[3] = -1.0
    rc, st = _host_call(plan, x, y, good, r_bad, out)
    assert rc == _native.ENKF_INVALID_ARGUMENT and b"positive" in st.message
    x_nan = x.copy()
    x_nan[good[17], 3] = np.nan
    rc, st = _host_call(plan, x_nan, y, good, r, out)
    assert rc == _native.ENKF_INVALID_ARGUMENT and b"non-finite" in st.message
    rc, st = _host_call(plan, x, y, good, r, out)
    assert rc == 0, st.message
    assert rel_err(out, oracle.analysis_step(x, y, good, r)) <= 1e-9
