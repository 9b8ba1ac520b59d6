"""Parity of the CUDA path (libenkf_b200.so via the drop-in API / C ABI)
against the CPU oracle (oracle/) and the reference's golden fixtures.

Tolerances (written here, per the north star): the analysis ensemble X^A
within 1e-9 max-relative error (max|dX^A| / max|X^A_ref|, the reference's
own normwise convention); Z of solve_sherman within 1e-11 relative (the
reference tests' dense-solve bound is 1e-11 absolute, test_sherman.py:41-44).
"""

import ctypes

import numpy as np
import pytest

import oracle
from golden_io import ism_cases, kalman_cases, load, rel_err
import paper_1302_3876_b200 as P
from paper_1302_3876_b200 import _native
from paper_1302_3876_b200 import workloads as W

pytestmark = pytest.mark.gpu

XA_TOL = 1e-9
Z_TOL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1302_3876_b200.build import build
    build()
    import torch
    assert torch.cuda.is_available()


def obs_of(p):
    return P.ObservationBatch(y=p.y, perturbed=p.perturbed, perturbations=p.perturbed - p.y[:, None])


def h_of(p):
    return P.SelectionOperator.identity() if p.indices is None else P.SelectionOperator.from_indices(p.indices)


# ---------------------------------------------------------------- solve_sherman
@pytest.mark.parametrize("case", list(range(22)))
def test_solve_matches_reference_golden(case):
    seed, r, v, d, z_ref, zl_ref, ops = list(ism_cases())[case]
    res = P.solve_sherman(r, v, d, count_ops=True)
    assert isinstance(res.z, np.ndarray) and res.z.shape == z_ref.shape and res.z.flags.c_contiguous
    assert rel_err(res.z, z_ref) <= Z_TOL
    assert rel_err(res.z, zl_ref) <= Z_TOL
    assert res.long_ops == ops
    assert res.seconds > 0


def test_zero_v_is_diagonal_solve():
    z = P.solve_sherman(np.array([2.0, 2.0]), np.zeros((2, 1)), np.array([[4.0], [6.0]])).z
    assert np.array_equal(z, [[2.0], [3.0]])


def test_scalar_rank_one():
    z = P.solve_sherman(np.array([1.0]), np.array([[1.0]]), np.array([[1.0]])).z
    assert np.allclose(z, [[0.5]], atol=1e-15)


def test_against_dense_solve():
    g = np.random.Generator(np.random.Philox(31))
    r = g.uniform(0.5, 2.0, 5)
    v = g.standard_normal((5, 3))
    d = g.standard_normal((5, 3))
    z = P.solve_sherman(r, v, d).z
    assert np.abs(z - np.linalg.solve(np.diag(r) + v @ v.T, d)).max() <= 1e-11


@pytest.mark.parametrize("nobs,nens", [(50, 2), (200, 16), (2000, 128), (70000, 128), (333, 77)])
def test_residual_bound(nobs, nens):
    g = np.random.Generator(np.random.Philox(40 + nens))
    r = g.uniform(0.5, 2.0, nobs)
    v = g.standard_normal((nobs, nens))
    d = g.standard_normal((nobs, nens))
    z = P.solve_sherman(r, v, d).z
    residual = np.abs(r[:, None] * z + v @ (v.T @ z) - d).max()
    bound = 1e-10 * (np.abs(d).max() + np.abs(v).sum(axis=1).max() ** 2 * np.abs(z).max())
    assert residual <= bound


def test_validation_errors():
    with pytest.raises(ValueError):
        P.solve_sherman(np.array([1.0, 1.0]), np.ones((3, 2)), np.ones((3, 2)))
    with pytest.raises(ValueError):
        P.solve_sherman(np.array([1.0, -1.0]), np.ones((2, 2)), np.ones((2, 2)))
    with pytest.raises(ValueError):
        P.solve_sherman(np.array([1.0, 1.0]), np.ones((2, 2)), np.ones((2, 3)))
    bad = np.ones((2, 2))
    bad[0, 0] = np.inf
    with pytest.raises(ValueError):
        P.solve_sherman(np.array([1.0, 1.0]), bad, np.ones((2, 2)))
    # empty observation set: the reference's sweep raises ValueError (sherman.py:187)
    with pytest.raises(ValueError):
        P.solve_sherman(np.zeros(0), np.zeros((0, 3)), np.zeros((0, 3)))


def test_device_flags_non_finite_and_nonpositive():
    import torch
    dev = torch.device("cuda", 0)
    v = torch.ones((4, 2), dtype=torch.float64, device=dev)
    d = torch.ones((4, 2), dtype=torch.float64, device=dev)
    d[2, 1] = float("nan")
    with pytest.raises(ValueError):
        P.solve_sherman(torch.ones(4, dtype=torch.float64, device=dev), v, d)
    with pytest.raises(ValueError):
        P.solve_sherman(torch.tensor([1.0, 1.0, 0.0, 1.0], dtype=torch.float64, device=dev), v, torch.ones_like(v))


@pytest.mark.parametrize("maker", ["config1", "config4s10"])
def test_device_resident_r_validated_on_device(maker):
    """A CUDA-tensor r is not copied back for validation: r <= 0 and non-finite r are
    flagged by the Gram pass and raise the reference's ValueError (sherman.py:100-107)."""
    import torch
    p = {"config1": W.config1, "config4s10": lambda: W.config4(10)}[maker]()
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(p.x).to(dev)
    obs = P.ObservationBatch(y=None, perturbed=torch.from_numpy(p.perturbed).to(dev), perturbations=None)
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        r = torch.from_numpy(p.r).to(dev)
        r[len(p.r) // 2] = bad
        with pytest.raises(ValueError):
            P.analysis_step(x, obs, h_of(p), r)
    xa = P.analysis_step(x, obs, h_of(p), torch.from_numpy(p.r).to(dev))
    assert rel_err(xa.cpu().numpy(), oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)) <= XA_TOL


def _levels_on(gram_host, n):
    import torch
    dev = torch.device("cuda", 0)
    plan = _native.Plan(0, 4, n, 0)
    lib = _native.lib()
    g = torch.as_tensor(gram_host, dtype=torch.float64, device=dev).contiguous()
    a = torch.empty((n, n), dtype=torch.float64, device=dev)
    den = torch.empty(n, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    assert lib.enkf_plan_reset_status(plan.handle, s) == 0
    assert lib.enkf_ism_levels_f64(plan.handle, g.data_ptr(), a.data_ptr(), None, den.data_ptr(), s) == 0
    st = _native.EnkfStatus()
    code = lib.enkf_plan_sync_status(plan.handle, s, ctypes.byref(st))
    return code, st, a.cpu().numpy(), den.cpu().numpy()


def test_singular_update_guard_reports_level():
    # the unvalidated core (test_sherman.py:67-77): r = -1, v = d = 1 gives
    # den_1 = 1 + v'u = 1 + 1/(-1) = 0 at level 1
    code, st, _, _ = _levels_on(np.array([[-1.0, -1.0]]), 1)
    assert code == _native.ENKF_SINGULAR_UPDATE and st.level == 1 and abs(st.denominator) < 1e-14
    with pytest.raises(P.SingularUpdateError) as info:
        _native.raise_for_status(code, st)
    assert info.value.level == 1
    g = np.zeros((3, 6))
    g[0, 0], g[1, 1], g[2, 2] = 0.5, 2.0, -1.0
    code, st, _, den = _levels_on(g, 3)
    assert code == _native.ENKF_SINGULAR_UPDATE and st.level == 3


def test_levels_match_model():
    import reduced_model as M
    for _, r, v, d, *_ in list(ism_cases())[:6]:
        g = M.gram_solve(v, d, r)
        code, st, a, den = _levels_on(g, v.shape[1])
        a_m, den_m = M.levels(g)
        assert code == 0
        assert rel_err(a, a_m) <= 1e-12 and rel_err(den, den_m) <= 1e-13


# ---------------------------------------------------------------- analysis_step
def test_kalman_gain_instances_match_reference():
    for x, idx, r, perturbed, xa_ref in kalman_cases():
        h = P.SelectionOperator.from_indices(idx)
        obs = P.ObservationBatch(y=perturbed[:, 0], perturbed=perturbed, perturbations=perturbed * 0)
        xa = P.analysis_step(x, obs, h, r, "sherman")
        assert np.abs(xa - xa_ref).max() <= 1e-12 * max(1.0, np.abs(xa_ref).max())
        s = oracle.member_deviations(x)
        hm = np.zeros((idx.size, x.shape[0]))
        hm[np.arange(idx.size), idx] = 1.0
        p = s @ s.T
        gain = p @ hm.T @ np.linalg.inv(hm @ p @ hm.T + np.diag(r))
        assert np.abs(xa - (x + gain @ (perturbed - hm @ x))).max() <= 1e-9


def test_zero_spread_is_identity():
    x = np.tile(np.arange(6.0)[:, None], (1, 4))
    h = P.SelectionOperator.from_indices([1, 4])
    obs = P.ObservationBatch(y=np.array([5.0, -2.0]), perturbed=np.array([[5.0] * 4, [-2.0] * 4]),
                             perturbations=np.zeros((2, 4)))
    xa = P.analysis_step(x, obs, h, np.ones(2), "sherman")
    assert np.array_equal(xa, x)


def test_uninformative_observations():
    g = np.random.Generator(np.random.Philox(1))
    x = g.standard_normal((10, 4))
    idx = np.sort(g.choice(10, size=6, replace=False))
    y = g.standard_normal(6)
    obs = P.ObservationBatch(y=y, perturbed=y[:, None] + 0.2 * g.standard_normal((6, 4)), perturbations=None)
    xa = P.analysis_step(x, obs, P.SelectionOperator.from_indices(idx), np.full(6, 1e12), "sherman")
    assert np.abs(xa - x).max() <= 1e-6 * np.abs(x).max()


def test_returns_new_array_inputs_untouched():
    p = W.config1()
    x0, y0 = p.x.copy(), p.perturbed.copy()
    xa = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
    assert not np.shares_memory(xa, p.x) and xa.flags.c_contiguous and xa.dtype == np.float64
    assert np.array_equal(p.x, x0) and np.array_equal(p.perturbed, y0)


def test_config1_golden():
    g = load("configs")
    h = P.SelectionOperator.from_indices(g["c1_idx"])
    obs = P.ObservationBatch(y=None, perturbed=g["c1_perturbed"], perturbations=None)
    xa = P.analysis_step(g["c1_x"], obs, h, g["c1_r"])
    assert rel_err(xa, g["c1_xa"]) <= XA_TOL


@pytest.mark.parametrize("tag", ["c2", "c3", "c4s8"])
def test_config_goldens(tag):
    g = load("configs")
    p = {"c2": lambda: W.Config2Cycler().cycle(), "c3": W.config3, "c4s8": lambda: W.config4(8)}[tag]()
    xa = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
    stride = int(g[f"{tag}_stride"])
    assert rel_err(xa[::stride], g[f"{tag}_xa_rows"]) <= XA_TOL
    assert np.abs(xa.sum(axis=0) - g[f"{tag}_xa_colsum"]).max() <= 1e-9 * xa.shape[0] * float(g[f"{tag}_xa_absmax"])


@pytest.mark.parametrize("maker", ["config1", "config3", "config4s6", "config4s4", "config5s6"])
def test_analysis_vs_oracle(maker):
    p = {"config1": W.config1, "config3": W.config3, "config4s6": lambda: W.config4(6),
         "config4s4": lambda: W.config4(4), "config5s6": lambda: W.config5(6)}[maker]()
    xa = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
    ref = oracle.analysis_step_chunked(p.x, p.perturbed, p.indices, p.r)
    err = rel_err(xa, ref)
    print(f"{maker}: X^A rel err vs oracle {err:.3e}")
    assert err <= XA_TOL


@pytest.mark.parametrize("case", list(range(16)))
def test_random_systems_analysis(case):
    """Acceptance-C1-style sweep (test_acceptance.py:44-61) on the whole analysis step:
    random ensemble sizes 2..128 (N = 128 takes the int8 tensor-core Gram and anomaly
    kernels, others the FP64 DMMA ones), n_obs log-uniform in 10..20000 (down to one
    partial 32-row block of the int8 Gram), random sorted H, value scales spanning
    decades; X^A against the oracle within 1e-9 and against the explicit Kalman gain."""
    g = np.random.Generator(np.random.Philox(9000 + case))
    n = int(g.choice([2, 3, 7, 20, 31, 64, 97, 128, 128, 128]))
    nobs = int(np.exp(g.uniform(np.log(10), np.log(20000))))
    ns = nobs + int(g.integers(0, 3 * nobs + 1))
    idx = np.sort(g.choice(ns, nobs, replace=False))
    scale = 10.0 ** g.uniform(-3, 3, ns)[:, None]
    x = scale * (g.standard_normal((ns, 1)) + g.uniform(0.2, 2.0) * g.standard_normal((ns, n)))
    r = (g.uniform(0.1, 2.0, nobs) * scale[idx, 0]) ** 2
    y = x[idx].mean(axis=1, keepdims=True) + np.sqrt(r)[:, None] * g.standard_normal((nobs, n))
    xa = P.analysis_step(x, P.ObservationBatch(y=None, perturbed=y, perturbations=None),
                         P.SelectionOperator.from_indices(idx), r)
    assert rel_err(xa, oracle.analysis_step(x, y, idx, r)) <= XA_TOL, (n, nobs, ns)
    # explicit gain X + P H'(H P H' + R)^-1 (Y - H X) (test_enkf.py:215-225)
    s = (x - x.mean(axis=1, keepdims=True)) / np.sqrt(n - 1)
    v = s[idx]
    k = s @ v.T @ np.linalg.inv(v @ v.T + np.diag(r)) if nobs <= 3000 else None
    if k is not None:
        assert rel_err(xa, x + k @ (y - x[idx])) <= 1e-8, (n, nobs, ns)


def test_config2_cycles_open_loop():
    """Config 2: all 100 assimilation cycles of the configuration, identical X^B to
    GPU and oracle at every cycle (open loop), the GPU analysis driving the next
    forecast."""
    cyc = W.Config2Cycler()
    xa = None
    for c in range(100):
        p = cyc.cycle(xa)
        xa = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
        assert rel_err(xa, oracle.analysis_step(p.x, p.perturbed, None, p.r)) <= XA_TOL, c


def test_device_resident_path_matches_host_path():
    import torch
    p = W.config4(8)
    dev = torch.device("cuda", 0)
    xa_h = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
    x = torch.from_numpy(p.x).to(dev)
    obs = P.ObservationBatch(y=None, perturbed=torch.from_numpy(p.perturbed).to(dev), perturbations=None)
    xa_d = P.analysis_step(x, obs, h_of(p), torch.from_numpy(p.r).to(dev))
    assert xa_d.is_cuda and xa_d.dtype == torch.float64
    assert np.array_equal(xa_d.cpu().numpy(), xa_h)


def test_run_to_run_bitwise_determinism():
    p = W.config4(6)
    a = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
    b = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
    assert np.array_equal(a, b)


def test_member_deviations_and_innovations():
    p = W.config3()
    s = P.member_deviations(p.x)
    assert rel_err(s, oracle.member_deviations(p.x)) <= 1e-14
    d = P.innovations(obs_of(p), h_of(p), p.x)
    assert np.array_equal(d, oracle.innovations(p.perturbed, p.indices, p.x))


def test_device_index_errors_flagged():
    """Device idx out of range / unsorted is flagged by the Gram kernel (the C
    ABI's own guard; the Python layer validates before launch)."""
    import torch
    dev = torch.device("cuda", 0)
    n = 4
    plan = _native.Plan(8, 3, n, 0)
    x = torch.randn((8, n), dtype=torch.float64, device=dev)
    y = torch.randn((3, n), dtype=torch.float64, device=dev)
    r = torch.ones(3, dtype=torch.float64, device=dev)
    out = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    for bad, code in (([1, 5, 9], _native.ENKF_INDEX_RANGE), ([1, 5, 5], _native.ENKF_INVALID_ARGUMENT)):
        idx = torch.tensor(bad, dtype=torch.int64, device=dev)
        st = _native.EnkfStatus()
        rc = _native.lib().enkf_analysis_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(),
                                            r.data_ptr(), out.data_ptr(), s, ctypes.byref(st))
        assert rc == code, st.message


def _staged_analysis(plan, x, y, idx, r):
    import torch
    n = x.shape[1]
    dev = x.device
    gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
    a = torch.empty((n, n), dtype=torch.float64, device=dev)
    t = torch.empty((n, n), dtype=torch.float64, device=dev)
    out = torch.empty_like(x)
    lib = _native.lib()
    s = torch.cuda.current_stream().cuda_stream
    assert lib.enkf_plan_reset_status(plan.handle, s) == 0
    assert lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), 0 if idx is None else idx.data_ptr(),
                                 r.data_ptr(), gram.data_ptr(), s) == 0
    assert lib.enkf_ism_levels_f64(plan.handle, gram.data_ptr(), a.data_ptr(), t.data_ptr(), None, s) == 0
    assert lib.enkf_anomaly_update_f64(plan.handle, x.data_ptr(), t.data_ptr(), out.data_ptr(), x.shape[0], s) == 0
    st = _native.EnkfStatus()
    _native.raise_for_status(lib.enkf_plan_sync_status(plan.handle, s, ctypes.byref(st)), st)
    return gram.cpu().numpy(), out.cpu().numpy()


@pytest.mark.parametrize("maker", ["config4s8", "config3"])
def test_tma_kernels_match_generic_kernels(maker, monkeypatch):
    """The warp-specialised TMA kernels (production) and the generic cp.async
    kernels (odd N / unaligned fallback) agree."""
    import torch
    p = {"config4s8": lambda: W.config4(8), "config3": W.config3}[maker]()
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(p.x).to(dev)
    y = torch.from_numpy(p.perturbed).to(dev)
    r = torch.from_numpy(p.r).to(dev)
    idx = None if p.indices is None else torch.from_numpy(p.indices).to(dev)
    ns, nobs, n = p.shape
    plan_ws = _native.Plan(ns, nobs, n, 0)             # N == 128: gram128 kernel
    monkeypatch.setenv("ENKF_DISABLE_G128", "1")
    plan_ws_gen = _native.Plan(ns, nobs, n, 0)         # general warp-specialised kernel
    monkeypatch.setenv("ENKF_DISABLE_WS", "1")
    plan_gen = _native.Plan(ns, nobs, n, 0)            # cp.async fallback kernels
    g1, xa1 = _staged_analysis(plan_ws, x, y, idx, r)
    g2, xa2 = _staged_analysis(plan_gen, x, y, idx, r)
    g3, xa3 = _staged_analysis(plan_ws_gen, x, y, idx, r)
    assert rel_err(g1, g2) <= 1e-13 and rel_err(g3, g2) <= 1e-13
    assert rel_err(xa1, xa2) <= 1e-12 and rel_err(xa3, xa2) <= 1e-12
    ref = oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)
    assert rel_err(xa1, ref) <= XA_TOL and rel_err(xa2, ref) <= XA_TOL


@pytest.mark.parametrize("ws", ["0", "1"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8, 16, 20, 33, 50, 64, 66, 96, 100, 127, 128])
def test_solve_ensemble_size_sweep(n, ws, monkeypatch):
    """Every ensemble size up to the maximum, through both kernel families
    (TMA/warp-specialised for even N, generic cp.async otherwise)."""
    import torch
    import reduced_model as M
    monkeypatch.setenv("ENKF_DISABLE_WS", ws)
    dev = torch.device("cuda", 0)
    lib = _native.lib()
    s = torch.cuda.current_stream().cuda_stream
    for nobs in (5, 50, 1000):
        g = np.random.Generator(np.random.Philox(n * 1000 + nobs))
        r = g.uniform(0.5, 2, nobs)
        v = g.standard_normal((nobs, n))
        d = g.standard_normal((nobs, n))
        plan = _native.Plan(0, nobs, n, 0)
        z = torch.empty((nobs, n), dtype=torch.float64, device=dev)
        a = torch.empty((n, n), dtype=torch.float64, device=dev)
        rt, vt, dt = (torch.from_numpy(t).to(dev) for t in (r, v, d))
        st = _native.EnkfStatus()
        rc = lib.enkf_ism_solve_f64(plan.handle, rt.data_ptr(), vt.data_ptr(), dt.data_ptr(), z.data_ptr(),
                                    a.data_ptr(), s, ctypes.byref(st))
        assert rc == 0, st.message
        zm, am = M.solve(r, v, d)
        assert rel_err(z.cpu().numpy(), zm) <= 1e-11, (n, nobs)
        assert rel_err(a.cpu().numpy(), am) <= 1e-10, (n, nobs)
        z_or, _ = oracle.solve_sherman(r, v, d)
        assert rel_err(z.cpu().numpy(), z_or) <= Z_TOL, (n, nobs)


@pytest.mark.parametrize("maker", ["config4s8", "config4s4", "config5s6"])
def test_tensor_core_anomaly_matches_fp64(maker, monkeypatch):
    """The int8-digit tcgen05 anomaly update (default for N = 128) against the
    FP64 DMMA kernel and the oracle: fp64-grade (<= 1e-12 relative to max|X^A|)."""
    import torch
    p = {"config4s8": lambda: W.config4(8), "config4s4": lambda: W.config4(4),
         "config5s6": lambda: W.config5(6)}[maker]()
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(p.x).to(dev)
    y = torch.from_numpy(p.perturbed).to(dev)
    r = torch.from_numpy(p.r).to(dev)
    idx = torch.from_numpy(p.indices).to(dev)
    ns, nobs, n = p.shape
    assert n == 128
    plan_tc = _native.Plan(ns, nobs, n, 0)
    monkeypatch.setenv("ENKF_ANOMALY", "fp64")
    plan_f64 = _native.Plan(ns, nobs, n, 0)
    _, xa_tc = _staged_analysis(plan_tc, x, y, idx, r)
    _, xa_f64 = _staged_analysis(plan_f64, x, y, idx, r)
    err = rel_err(xa_tc, xa_f64)
    print(f"{maker}: tcgen05-int8 vs fp64 DMMA {err:.2e}")
    assert err <= 1e-12
    ref = oracle.analysis_step_chunked(p.x, p.perturbed, p.indices, p.r)
    assert rel_err(xa_tc, ref) <= XA_TOL


def test_plan_options_select_the_kernels(monkeypatch):
    """enkf_plan_create_ex: the kernel families are plan parameters of the C ABI (the
    ENKF_* environment variables only set process-wide defaults).  A plan created with
    {gram_kernel: FP64, anomaly_kernel: FP64} computes bit for bit what a plan created
    under ENKF_GRAM=fp64 ENKF_ANOMALY=fp64 computes, the single-CTA levels option what
    the cluster kernel computes, and all of them agree with the default int8-digit
    plan to fp64 rounding level."""
    import torch
    p = W.config4(8)
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(p.x).to(dev)
    y = torch.from_numpy(p.perturbed).to(dev)
    r = torch.from_numpy(p.r).to(dev)
    idx = torch.from_numpy(p.indices).to(dev)
    ns, nobs, n = p.shape
    for k in ("ENKF_GRAM", "ENKF_ANOMALY", "ENKF_LEVELS"):
        monkeypatch.delenv(k, raising=False)
    plan_def = _native.Plan(ns, nobs, n, 0)
    assert (plan_def.options.gram_kernel, plan_def.options.anomaly_kernel) == (0, 0)
    plan_opt = _native.Plan(ns, nobs, n, 0, options={"gram_kernel": 1, "anomaly_kernel": 1})
    plan_lv = _native.Plan(ns, nobs, n, 0, options={"levels_kernel": 1})
    monkeypatch.setenv("ENKF_GRAM", "fp64")
    monkeypatch.setenv("ENKF_ANOMALY", "fp64")
    plan_env = _native.Plan(ns, nobs, n, 0)
    assert (plan_env.options.gram_kernel, plan_env.options.anomaly_kernel) == (1, 1)
    _, xa_def = _staged_analysis(plan_def, x, y, idx, r)
    _, xa_opt = _staged_analysis(plan_opt, x, y, idx, r)
    _, xa_env = _staged_analysis(plan_env, x, y, idx, r)
    _, xa_lv = _staged_analysis(plan_lv, x, y, idx, r)
    assert np.array_equal(xa_opt, xa_env)
    assert np.array_equal(xa_lv, xa_def)
    assert not np.array_equal(xa_opt, xa_def)       # different kernels did run
    assert rel_err(xa_def, xa_opt) <= 1e-11


def test_tensor_core_anomaly_zero_spread_and_nonfinite():
    import torch
    dev = torch.device("cuda", 0)
    n, ns = 128, 1000
    g = np.random.Generator(np.random.Philox(5))
    x = np.tile(g.standard_normal(ns)[:, None], (1, n))     # zero spread
    idx = np.arange(0, ns, 7)
    y = x[idx] + 0.3
    xa = P.analysis_step(x, P.ObservationBatch(y=None, perturbed=y, perturbations=None),
                         P.SelectionOperator.from_indices(idx), np.ones(idx.size))
    assert np.array_equal(xa, x)                              # exact, as in the reference
    # a non-finite unobserved row propagates (NaN row), finite rows are unaffected
    x2 = g.standard_normal((ns, n))
    x2[3, 5] = np.inf
    plan = _native.Plan(ns, idx.size, n, 0)
    xt = torch.from_numpy(x2).to(dev)
    t = torch.eye(n, dtype=torch.float64, device=dev) + 0.01
    out = torch.empty_like(xt)
    s = torch.cuda.current_stream().cuda_stream
    assert _native.lib().enkf_anomaly_update_f64(plan.handle, xt.data_ptr(), t.data_ptr(), out.data_ptr(), ns, s) == 0
    o = out.cpu().numpy()
    assert np.isnan(o[3]).all()
    mask = np.ones(ns, bool)
    mask[3] = False
    ref = x2[mask] @ t.cpu().numpy()
    assert rel_err(o[mask], ref) <= 1e-12


# ---------------------------------------------------------------- opt-in int8 Gram
def _gram_with(mode, heavy=False, ns_log2=17, no_log2=15):
    import os
    import subprocess
    import sys
    code = r'''
import os, sys, ctypes
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1302_3876_b200 import _native
heavy = int(sys.argv[1])
dev = torch.device("cuda", 0); lib = _native.lib(); s = torch.cuda.current_stream().cuda_stream
n, ns, no = 128, 1 << int(sys.argv[3]), 1 << int(sys.argv[4])
g = torch.Generator(device=dev); g.manual_seed(11)
x = torch.randn((ns, 1), dtype=torch.float64, device=dev, generator=g) + (0.5 + 1.5 * torch.rand((ns, 1), dtype=torch.float64, device=dev, generator=g)) * torch.randn((ns, n), dtype=torch.float64, device=dev, generator=g)
idx = torch.sort(torch.randperm(ns, device=dev, generator=g)[:no]).values
y = x[idx].mean(dim=1, keepdim=True) + torch.randn((no, n), dtype=torch.float64, device=dev, generator=g)
if heavy == 1:
    y[no // 3, 5] = 1e6
if heavy == 2:
    # an element whose 48-bit value sits just below 2^47 of its column scale, where
    # V + bias no longer fits six balanced digits: must take the overflow route
    e = (0.2 * torch.randn((no, n), dtype=torch.float64, device=dev, generator=g)).clamp(-0.2, 0.2)
    e[::16, :] = 0.25
    e[::16, 5] = 1.0
    e[17, 5] = 7.99
    y = x[idx] + e
r = 0.25 + 0.75 * torch.rand((no,), dtype=torch.float64, device=dev, generator=g)
if heavy == 2:
    r = torch.ones((no,), dtype=torch.float64, device=dev)
plan = _native.Plan(ns, no, n, 0)
gram = torch.empty((n, 2 * n), dtype=torch.float64, device=dev)
assert lib.enkf_ism_gram_f64(plan.handle, x.data_ptr(), y.data_ptr(), idx.data_ptr(), r.data_ptr(), gram.data_ptr(), s) == 0
st = _native.EnkfStatus()
assert lib.enkf_plan_sync_status(plan.handle, s, ctypes.byref(st)) == 0
np.save(sys.argv[2], gram.cpu().numpy())
'''
    import tempfile
    out = tempfile.mktemp(suffix=".npy")
    env = dict(os.environ, ENKF_GRAM=mode)
    subprocess.run([sys.executable, "-c", code, str(int(heavy)), out, str(ns_log2), str(no_log2)], env=env,
                   check=True, timeout=300)
    return np.load(out)


@pytest.mark.parametrize("mode", ["i8ls"])
@pytest.mark.parametrize("heavy", [0, 1, 2])
def test_int8_gram_matches_fp64_gram(heavy, mode):
    """The exact-digit tcgen05 Gram (default for N = 128) agrees with the FP64 DMMA
    Gram (ENKF_GRAM=fp64) to rounding level; a heavy-tailed element outside the
    sampled scales (1), or one at the top edge of the digit range (2), takes the
    device-gated FP64 fallback (then the two are identical).  "i8ls" is the default
    two-kernel form (slice pass + level-split MMA pass: N = 256 MMAs, A from shared
    memory)."""
    a, b = _gram_with("fp64", heavy), _gram_with(mode, heavy)
    assert np.abs(b[:, :128] - b[:, :128].T).max() == 0.0
    tol = 0.0 if heavy else 1e-13
    assert np.abs(a - b).max() <= tol * np.abs(a).max()


def test_int8_gram_level_split_mid_size():
    """2^20 observation rows: ~886 blocks per group of the level-split MMA pass, so
    the producers' pacing (a CTA more than G8LS_LEAD = 48 blocks ahead of its group
    polls the group's progress) and the multi-period flush (every 512 blocks) both
    run; agrees with the FP64 Gram to rounding level, exactly symmetric."""
    a, b = _gram_with("fp64", 0, 21, 20), _gram_with("i8ls", 0, 21, 20)
    assert np.abs(b[:, :128] - b[:, :128].T).max() == 0.0
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


@pytest.mark.parametrize("n", [2, 5, 8, 20, 31, 64, 96, 97, 127, 128])
def test_levels_cluster_equals_single_cta(n, monkeypatch):
    """The N Sherman-Morrison levels on a 4-CTA cluster (default; V'V columns and V'D
    bands split over the CTAs, pivot columns exchanged through distributed shared
    memory) perform the single-CTA kernel's arithmetic in the same order: A, T and
    every den_k agree bit for bit, and A matches a dense solve of (I + V'V) A = V'D."""
    import torch
    dev = torch.device("cuda", 0)
    g = np.random.Generator(np.random.Philox(40 + n))
    v = g.standard_normal((3000, n)) / np.sqrt(max(n - 1, 1))
    d = g.standard_normal((3000, n))
    gram = np.concatenate([v.T @ v, v.T @ d / np.sqrt(max(n - 1, 1))], axis=1)
    gd = torch.from_numpy(gram).to(dev)
    s = torch.cuda.current_stream().cuda_stream
    out = {}
    for mode in ("single", "cluster"):
        monkeypatch.setenv("ENKF_LEVELS", mode)
        plan = _native.Plan(1, 1, n, 0)
        a = torch.full((n, n), float("nan"), dtype=torch.float64, device=dev)
        t = torch.full_like(a, float("nan"))
        den = torch.full((n,), float("nan"), dtype=torch.float64, device=dev)
        assert _native.lib().enkf_plan_reset_status(plan.handle, s) == 0
        assert _native.lib().enkf_ism_levels_f64(plan.handle, gd.data_ptr(), a.data_ptr(), t.data_ptr(),
                                                 den.data_ptr(), s) == 0
        st = _native.EnkfStatus()
        assert _native.lib().enkf_plan_sync_status(plan.handle, s, ctypes.byref(st)) == 0, st.message
        out[mode] = (a.cpu().numpy(), t.cpu().numpy(), den.cpu().numpy())
    monkeypatch.delenv("ENKF_LEVELS")
    for k in range(3):
        assert np.array_equal(out["single"][k], out["cluster"][k]), (n, k)
    ref = np.linalg.solve(np.eye(n) + gram[:, :n], gram[:, n:])
    assert np.abs(out["cluster"][0] - ref).max() <= 1e-12 * np.abs(ref).max()


def test_levels_cluster_singular_level(monkeypatch):
    """The singular guard (sherman.py:171-174) on the cluster kernel: the first failing
    1-based level and its denominator, as the single-CTA kernel reports them."""
    import torch
    dev = torch.device("cuda", 0)
    n = 40
    gram = np.zeros((n, 2 * n))
    gram[:, :n] = np.eye(n)
    gram[17, 17] = -1.0  # den_18 = 1 + (-1) = 0
    gd = torch.from_numpy(gram).to(dev)
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    for mode in ("single", "cluster"):
        monkeypatch.setenv("ENKF_LEVELS", mode)
        plan = _native.Plan(1, 1, n, 0)
        a = torch.empty((n, n), dtype=torch.float64, device=dev)
        _native.lib().enkf_plan_reset_status(plan.handle, s)
        _native.lib().enkf_ism_levels_f64(plan.handle, gd.data_ptr(), a.data_ptr(), None, None, s)
        st = _native.EnkfStatus()
        code = _native.lib().enkf_plan_sync_status(plan.handle, s, ctypes.byref(st))
        res[mode] = (code, st.level, st.denominator)
    monkeypatch.delenv("ENKF_LEVELS")
    assert res["cluster"] == res["single"] and res["cluster"][0] == _native.ENKF_SINGULAR_UPDATE
    assert res["cluster"][1] == 18


def test_anomaly_debug_env_has_no_effect(monkeypatch):
    """The profiling role skips of anomaly_i8_kernel are compiled out of the product
    library: ENKF_I8_DBG set at plan creation changes nothing (bitwise)."""
    p = W.config4(8)
    base = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
    _native._plans.clear()
    monkeypatch.setenv("ENKF_I8_DBG", "7")
    try:
        other = P.analysis_step(p.x, obs_of(p), h_of(p), p.r)
    finally:
        monkeypatch.delenv("ENKF_I8_DBG")
        _native._plans.clear()
    assert np.array_equal(base, other)


@pytest.mark.parametrize("workers", [1, 2, 4, 8])
def test_solve_analysis_dispatch_and_blocked_workers(workers):
    """solvers.py:91-112 on the GPU: solve_analysis("sherman", ..., workers) runs
    solve_sherman (workers = 1) or solve_sherman_blocked (workers > 1, sherman.py:289-311);
    every worker count gives the bitwise-same Z as solve_sherman (the reference's
    tests/test_sherman.py:134-146 asserts workers=1 bitwise and the rest within 1e-12),
    and the result matches the reference's golden Z."""
    seed, r, v, d, z_ref, zl_ref, ops = list(ism_cases())[5]
    base = P.solve_sherman(r, v, d).z
    res = P.solve_analysis("sherman", r, v, d, workers=workers)
    assert isinstance(res, P.SolverResult)
    assert np.array_equal(res.z, base)
    assert np.array_equal(P.solve_sherman_blocked(r, v, d, workers=workers).z, base)
    assert np.array_equal(P.solve_analysis(P.SolverChoice.SHERMAN, r, v, d, workers=workers).z, base)
    assert rel_err(res.z, z_ref) <= Z_TOL


def test_solve_analysis_dispatch_errors():
    """Unknown names raise ValueError, the CPU baselines NotImplementedError
    (tests/test_solvers.py:111-129 pass-through / unknown-name behaviour)."""
    seed, r, v, d, *_ = list(ism_cases())[0]
    with pytest.raises(ValueError):
        P.solve_analysis("nope", r, v, d)
    for name in ("cholesky", "svd"):
        with pytest.raises(NotImplementedError):
            P.solve_analysis(name, r, v, d)
    with pytest.raises(ValueError):
        P.solve_sherman_blocked(r, v, d, workers=0)


def test_tensor_core_anomaly_extreme_rows():
    """Rows far from unit scale go through the same exact-digit path: tiny rows
    (max|x| < 2^-977: rescaled by 2^600 before slicing), huge rows (|x| ~ 1e300, the
    exponent-field slow path), all-zero rows and ordinary rows, one launch; each
    row against an fp64 X T computed on the host, relative to that row's scale.
    (Rows entirely in the subnormal range keep only the few bits fp64 has there.)"""
    import torch
    dev = torch.device("cuda", 0)
    n, ns = 128, 4096
    g = np.random.Generator(np.random.Philox(17))
    x = g.standard_normal((ns, n))
    scales = np.ones(ns)
    scales[0:64] = 2.0 ** -1000    # tiny
    scales[64:128] = 1e300         # huge (|X T| stays finite: T ~ I)
    scales[128:192] = 2.0 ** -990   # tiny, another binade
    x *= scales[:, None]
    x[192:256] = 0.0               # zero rows
    t = np.eye(n) + 0.02 * g.standard_normal((n, n))
    plan = _native.Plan(ns, 1, n, 0)
    xd = torch.from_numpy(x).to(dev)
    td = torch.from_numpy(t).to(dev)
    out = torch.empty_like(xd)
    s = torch.cuda.current_stream().cuda_stream
    assert _native.lib().enkf_anomaly_update_f64(plan.handle, xd.data_ptr(), td.data_ptr(), out.data_ptr(), ns, s) == 0
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    # reference in scaled arithmetic (x / scale) T, so the host product itself neither
    # underflows nor overflows
    safe = np.where(scales > 0, scales, 1.0)
    want = ((x / safe[:, None]) @ t) * safe[:, None]
    assert np.array_equal(got[192:256], np.zeros((64, n)))
    for lo, hi, tol in ((0, 64, 1e-12), (64, 128, 1e-12), (128, 192, 1e-12), (256, ns, 1e-12)):
        rowscale = np.abs(want[lo:hi]).max(axis=1, keepdims=True)
        assert np.all(np.isfinite(got[lo:hi]))
        assert (np.abs(got[lo:hi] - want[lo:hi]) / rowscale).max() <= tol, (lo, hi)


@pytest.mark.parametrize("n,nobs,ns", [(2, 3, 5), (5, 17, 40), (20, 20, 40), (33, 100, 300), (64, 512, 1024),
                                       (20, 40, 40)])
def test_tiny_path_equals_multi_kernel_path(n, nobs, ns, monkeypatch):
    """Desk-scale problems take the one-CTA kernel (tiny.cuh); it agrees with the
    multi-kernel path (ENKF_TINY=0) to rounding, in place (XA = X) and out of place,
    and keeps the index / validation errors."""
    import torch
    dev = torch.device("cuda", 0)
    g = np.random.Generator(np.random.Philox(500 + n + nobs))
    x = g.standard_normal((ns, 1)) + g.uniform(0.3, 2.0) * g.standard_normal((ns, n))
    idx = None if nobs == ns else np.sort(g.choice(ns, nobs, replace=False)).astype(np.int64)
    r = g.uniform(0.2, 1.5, nobs)
    y = (x if idx is None else x[idx]).mean(axis=1, keepdims=True) + g.standard_normal((nobs, n))
    xd, yd, rd = (torch.from_numpy(a).to(dev) for a in (x, y, r))
    idd = None if idx is None else torch.from_numpy(idx).to(dev)
    s = torch.cuda.current_stream().cuda_stream

    def run(tiny, inplace=False):
        monkeypatch.setenv("ENKF_TINY", "1" if tiny else "0")
        plan = _native.Plan(ns, nobs, n, 0)
        monkeypatch.delenv("ENKF_TINY")
        xin = xd.clone()
        out = xin if inplace else torch.empty_like(xd)
        st = _native.EnkfStatus()
        rc = _native.lib().enkf_analysis_f64(plan.handle, xin.data_ptr(), yd.data_ptr(),
                                            0 if idd is None else idd.data_ptr(), rd.data_ptr(), out.data_ptr(), s,
                                            ctypes.byref(st))
        assert rc == 0, st.message
        return out.cpu().numpy()

    a, b, c = run(True), run(False), run(True, inplace=True)
    assert rel_err(a, b) <= 1e-13
    assert np.array_equal(a, c)
    assert rel_err(a, oracle.analysis_step(x, y, idx, r)) <= XA_TOL
    if idx is not None and nobs > 2:  # the index checks of the Gram pass hold in the tiny kernel
        bad = idd.clone()
        bad[1] = bad[0]
        plan = _native.Plan(ns, nobs, n, 0)
        st = _native.EnkfStatus()
        rc = _native.lib().enkf_analysis_f64(plan.handle, xd.data_ptr(), yd.data_ptr(), bad.data_ptr(),
                                            rd.data_ptr(), torch.empty_like(xd).data_ptr(), s, ctypes.byref(st))
        assert rc == _native.ENKF_INVALID_ARGUMENT
