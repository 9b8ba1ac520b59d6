"""Localized analysis (enkf.py:193-199) and influence_matrix_cyclic
(enkf.py:138-164): CPU checks of the oracle and the host-side influence object
against the reference's golden fixture, and GPU parity of the localized-update
kernel (dense influence matrix and the matrix-free cyclic taper).

Tolerances: X^A within 1e-12 max-relative of the reference's output on the
small fixtures (the reference's own componentwise test uses 1e-12,
test_enkf.py:235-252); unit influence equals the unlocalized step within 1e-13
(test_enkf.py:254-260); 1e-11 against the oracle at larger sizes.
"""

import numpy as np
import pytest

import oracle
from golden_io import load, localized_cases, make_rng, rel_err
import paper_1302_3876_b200 as P

CASES = list(localized_cases())


def _h(idx):
    return P.SelectionOperator.identity() if idx is None else P.SelectionOperator.from_indices(idx)


def _obs(perturbed):
    return P.ObservationBatch(y=perturbed[:, 0], perturbed=perturbed, perturbations=perturbed - perturbed[:, :1])


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("i", range(len(CASES)))
def test_oracle_localized_matches_reference(i):
    c = CASES[i]
    xa = oracle.analysis_step_localized(c["x"], c["perturbed"], c["idx"], c["r"], c["delta"])
    assert rel_err(xa, c["xa"]) <= 1e-12


def test_oracle_and_package_influence_match_reference():
    g = load("localized")
    spec = {"i0": (10, [0, 5], None), "i1": (10, [5], None), "i2": (10, [9], None),
            "i3": (17, None, None), "i4": (10, [5], 2.0), "i5": (40, None, 8.0)}
    for tag, (ns, idx, sc) in spec.items():
        ref = g[f"{tag}_delta"]
        assert np.array_equal(oracle.influence_matrix_cyclic(ns, idx, sc), ref)
        lazy = P.influence_matrix_cyclic(ns, _h(idx), scale=sc)
        assert lazy.shape == ref.shape
        assert np.array_equal(np.asarray(lazy), ref)
    for c in CASES:
        if c["kind"] == "cyclic":
            lazy = P.influence_matrix_cyclic(c["x"].shape[0], _h(c["idx"]), scale=c["scale"])
            assert np.array_equal(np.asarray(lazy), c["delta"])


def test_influence_known_answers():
    # test_enkf.py:160-190
    d = P.influence_matrix_cyclic(10, P.SelectionOperator.from_indices([0, 5]))
    assert d[0, 0] == 1.0 and d[5, 1] == 1.0
    assert abs(P.influence_matrix_cyclic(10, P.SelectionOperator.from_indices([5]))[0, 0] - np.exp(-0.5)) <= 1e-12
    assert abs(P.influence_matrix_cyclic(10, P.SelectionOperator.from_indices([9]))[0, 0] - np.exp(-0.1)) <= 1e-12
    d = P.influence_matrix_cyclic(17, P.SelectionOperator.identity())
    assert d.min() > 0.0 and d.max() <= 1.0
    d = P.influence_matrix_cyclic(10, P.SelectionOperator.from_indices([5]), scale=2.0)
    assert abs(d[0, 0] - np.exp(-2.5)) <= 1e-12
    with pytest.raises(ValueError):
        P.influence_matrix_cyclic(10, P.SelectionOperator.identity(), scale=0.0)
    with pytest.raises(ValueError):
        P.influence_matrix_cyclic(10, P.SelectionOperator.from_indices([3, 12]))


def test_oracle_wrong_influence_shape():
    c = CASES[3]
    with pytest.raises(ValueError):
        oracle.analysis_step_localized(c["x"], c["perturbed"], c["idx"], c["r"], np.ones((3, 3)))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES)))
def test_gpu_localized_dense_matches_reference(i):
    c = CASES[i]
    xa = P.analysis_step(c["x"], _obs(c["perturbed"]), _h(c["idx"]), c["r"], "sherman", localization=c["delta"])
    assert isinstance(xa, np.ndarray) and xa.shape == c["x"].shape
    assert np.abs(xa - c["xa"]).max() <= 1e-12 * max(1.0, np.abs(c["xa"]).max())


@pytest.mark.gpu
@pytest.mark.parametrize("i", [k for k, c in enumerate(CASES) if c["kind"] == "cyclic"])
def test_gpu_localized_matrix_free_matches_reference(i):
    c = CASES[i]
    h = _h(c["idx"])
    lazy = P.influence_matrix_cyclic(c["x"].shape[0], h, scale=c["scale"])
    xa = P.analysis_step(c["x"], _obs(c["perturbed"]), h, c["r"], "sherman", localization=lazy)
    assert np.abs(xa - c["xa"]).max() <= 1e-12 * max(1.0, np.abs(c["xa"]).max())


@pytest.mark.gpu
def test_gpu_unit_influence_equals_unlocalized():
    c = CASES[3]
    h = _h(c["idx"])
    plain = P.analysis_step(c["x"], _obs(c["perturbed"]), h, c["r"], "sherman")
    loc = P.analysis_step(c["x"], _obs(c["perturbed"]), h, c["r"], "sherman",
                          localization=np.ones((c["x"].shape[0], c["r"].size)))
    assert np.abs(plain - loc).max() <= 1e-13 * max(1.0, np.abs(plain).max())


@pytest.mark.gpu
def test_gpu_componentwise_formula():
    # test_enkf.py:235-252 on the GPU
    rng = make_rng(4)
    x = rng.standard_normal((9, 4))
    idx = np.sort(rng.choice(9, size=5, replace=False))
    r = rng.uniform(0.2, 1.0, 5)
    pert = rng.standard_normal(5)[:, None] + 0.2 * rng.standard_normal((5, 4))
    delta = make_rng(44).uniform(0.0, 1.0, (9, 5))
    xa = P.analysis_step(x, _obs(pert), _h(idx), r, "sherman", localization=delta)
    s = oracle.member_deviations(x)
    v = s[idx]
    z, _ = oracle.solve_sherman(r, v, pert - x[idx])
    expected = x.copy()
    for i in range(9):
        for m in range(4):
            expected[i, m] += sum(s[i, k] * sum(delta[i, j] * v[j, k] * z[j, m] for j in range(5)) for k in range(4))
    assert np.abs(xa - expected).max() <= 1e-12 * max(1.0, np.abs(expected).max())


@pytest.mark.gpu
def test_gpu_wrong_influence_shape():
    c = CASES[3]
    with pytest.raises(ValueError):
        P.analysis_step(c["x"], _obs(c["perturbed"]), _h(c["idx"]), c["r"], "sherman", localization=np.ones((3, 3)))


@pytest.mark.gpu
@pytest.mark.parametrize("ns,nens,nobs,scale", [(4096, 64, 1024, 40.0), (3000, 128, None, 100.0),
                                                (1037, 33, 301, 7.5), (257, 2, 31, 3.0)])
def test_gpu_localized_vs_oracle_larger(ns, nens, nobs, scale):
    rng = make_rng(ns + nens)
    x = rng.standard_normal((ns, nens)) * rng.uniform(0.5, 2.0, (ns, 1)) + rng.standard_normal((ns, 1))
    idx = None if nobs is None else np.sort(rng.choice(ns, size=nobs, replace=False))
    m = ns if nobs is None else nobs
    r = rng.uniform(0.25, 1.0, m)
    pert = (x[idx] if idx is not None else x).mean(axis=1)[:, None] + rng.standard_normal((m, nens))
    h = _h(idx)
    lazy = P.influence_matrix_cyclic(ns, h, scale=scale)
    ref = oracle.analysis_step_localized(x, pert, idx, r, np.asarray(lazy))
    got_free = P.analysis_step(x, _obs(pert), h, r, "sherman", localization=lazy)
    got_dense = P.analysis_step(x, _obs(pert), h, r, "sherman", localization=np.asarray(lazy))
    assert rel_err(got_free, ref) <= 1e-11
    assert rel_err(got_dense, ref) <= 1e-11


@pytest.mark.gpu
def test_gpu_localized_device_resident_and_errors():
    import torch
    c = CASES[1]
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(c["x"]).to(dev)
    pert = torch.from_numpy(c["perturbed"]).to(dev)
    obs = P.ObservationBatch(y=pert[:, 0], perturbed=pert, perturbations=pert - pert[:, :1])
    h = _h(c["idx"])
    xa = P.analysis_step(x, obs, h, c["r"], "sherman", localization=torch.from_numpy(c["delta"]).to(dev))
    assert xa.is_cuda
    assert np.abs(xa.cpu().numpy() - c["xa"]).max() <= 1e-12 * max(1.0, np.abs(c["xa"]).max())
    with pytest.raises(ValueError):  # r <= 0, same ValueError as the unlocalized path
        P.analysis_step(c["x"], _obs(c["perturbed"]), h, -c["r"], "sherman", localization=c["delta"])
    bad = c["perturbed"].copy()
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        P.analysis_step(c["x"], _obs(bad), h, c["r"], "sherman", localization=c["delta"])


@pytest.mark.gpu
@pytest.mark.parametrize("nens", [5, 20, 64, 100, 128])
def test_gpu_localized_dmma_equals_cuda_core_form(nens, monkeypatch):
    """The DMMA localized update (default) and the CUDA-core form (ENKF_LOCALIZED=fma)
    agree to rounding on ragged sizes (state rows not a multiple of the 64-row CTA,
    observation count not a multiple of the 32-row chunk, N not a multiple of 8)."""
    import ctypes
    import torch
    from paper_1302_3876_b200 import _native
    rng = make_rng(77 + nens)
    ns, nobs = 1000, 333
    x = rng.standard_normal((ns, nens)) + rng.standard_normal((ns, 1))
    idx = np.sort(rng.choice(ns, size=nobs, replace=False)).astype(np.int64)
    r = rng.uniform(0.25, 1.0, nobs)
    pert = x[idx].mean(axis=1)[:, None] + rng.standard_normal((nobs, nens))
    dev = torch.device("cuda", 0)
    xd, yd, rd, idd = (torch.from_numpy(a).to(dev) for a in (x, pert, r, idx))
    outs = {}
    for mode in ("dmma", "fma"):
        if mode == "fma":
            monkeypatch.setenv("ENKF_LOCALIZED", "fma")
        plan = _native.Plan(ns, nobs, nens, 0)
        monkeypatch.delenv("ENKF_LOCALIZED", raising=False)
        out = torch.empty_like(xd)
        st = _native.EnkfStatus()
        rc = _native.lib().enkf_analysis_localized_cyclic_f64(
            plan.handle, xd.data_ptr(), yd.data_ptr(), idd.data_ptr(), rd.data_ptr(), 37.0, out.data_ptr(),
            torch.cuda.current_stream().cuda_stream, ctypes.byref(st))
        assert rc == 0, st.message
        outs[mode] = out.cpu().numpy()
    ref = oracle.analysis_step_localized(x, pert, idx, r, oracle.influence_matrix_cyclic(ns, idx, 37.0))
    assert rel_err(outs["dmma"], outs["fma"]) <= 1e-13
    assert rel_err(outs["dmma"], ref) <= 1e-11
