"""Pin the CPU oracle (oracle/) to the reference's own outputs (golden fixtures
produced by tests/golden/make_golden.py running /root/reference)."""

import numpy as np
import pytest

import oracle
from golden_io import ism_cases, kalman_cases, load, rel_err, sha
from paper_1302_3876_b200 import workloads as W


@pytest.mark.parametrize("case", list(range(22)))
def test_oracle_solve_matches_reference(case):
    seed, r, v, d, z_ref, zl_ref, ops_ref = list(ism_cases())[case]
    z, _ = oracle.solve_sherman(r, v, d)
    # same BLAS call sequence: bitwise on the host that made the fixtures,
    # BLAS-kernel rounding elsewhere
    assert rel_err(z, z_ref) <= 1e-13
    zl, ops = oracle.sweep_levelwise(r, v, d, count_ops=True)
    assert rel_err(zl, zl_ref) <= 1e-13
    assert ops == ops_ref == oracle.long_op_count(v.shape[1], v.shape[0])


def test_oracle_op_count_formula():
    for n, m, ops in load("ism_systems")["opcount"]:
        assert oracle.long_op_count(int(n), int(m)) == int(ops)
    with pytest.raises(ValueError):
        oracle.long_op_count(0, 5)


def test_oracle_kalman_instances():
    for x, idx, r, perturbed, xa_ref in kalman_cases():
        xa = oracle.analysis_step(x, perturbed, idx, r)
        assert rel_err(xa, xa_ref) <= 1e-13


def test_oracle_zero_spread():
    g = load("analysis_small")
    x = g["zero_x"]
    xa = oracle.analysis_step(x, np.array([[5.0] * 4, [-2.0] * 4]), np.array([1, 4]), np.ones(2))
    assert np.array_equal(xa, g["zero_xa"]) and np.array_equal(xa, x)


def test_config1_generator_and_oracle_match_reference():
    g = load("configs")
    p = W.config1()
    # our restated generator reproduces the reference-built inputs
    assert np.abs(p.x - g["c1_x"]).max() <= 1e-12
    assert np.array_equal(p.indices, g["c1_idx"])
    assert np.array_equal(p.r, g["c1_r"])
    assert np.abs(p.perturbed - g["c1_perturbed"]).max() <= 1e-12
    xa = oracle.analysis_step(g["c1_x"], g["c1_perturbed"], g["c1_idx"], g["c1_r"])
    assert rel_err(xa, g["c1_xa"]) <= 1e-13


@pytest.mark.parametrize("tag", ["c2", "c3", "c4s8"])
def test_oracle_configs_match_reference(tag):
    g = load("configs")
    p = {"c2": lambda: W.Config2Cycler().cycle(), "c3": W.config3, "c4s8": lambda: W.config4(8)}[tag]()
    assert sha(np.concatenate([p.x.ravel(), p.perturbed.ravel(), p.r])) == str(g[f"{tag}_input_sha"])
    xa = oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)
    stride = int(g[f"{tag}_stride"])
    assert rel_err(xa[::stride], g[f"{tag}_xa_rows"]) <= 1e-12
    assert np.abs(xa.sum(axis=0) - g[f"{tag}_xa_colsum"]).max() <= 1e-9 * xa.shape[0]


def test_chunked_oracle_matches_plain():
    p = W.config4(10)
    a = oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)
    b = oracle.analysis_step_chunked(p.x, p.perturbed, p.indices, p.r, rows_per_chunk=3000)
    assert rel_err(b, a) <= 1e-14


def test_identical_observation_selection():
    g = load("selection")
    assert np.array_equal(W.uniform_stride_indices(40, 0.5), g["c1"])
    assert W.uniform_stride_indices(4096, 1.0) is None and bool(g["c2_identity"])
    for sl in (8, 6):
        z, s = W.SIZES[4], W.SEEDS[4]
        ns, nobs = z["ns"] >> sl, z["nobs"] >> sl
        assert sha(W.random_indices(ns, nobs / ns, s["h"]).astype(np.int64)) == str(g[f"c4s{sl}_sha"])


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [4, 5])
def test_identical_observation_selection_full(cfg):
    g = load("selection")
    z, s = W.SIZES[cfg], W.SEEDS[cfg]
    idx = W.random_indices(z["ns"], z["nobs"] / z["ns"], s["h"]).astype(np.int64)
    assert idx.size == int(g[f"c{cfg}_n"])
    assert np.array_equal(idx[:512], g[f"c{cfg}_head"]) and np.array_equal(idx[-512:], g[f"c{cfg}_tail"])
    assert sha(idx) == str(g[f"c{cfg}_sha"])


def test_oracle_validation_errors():
    with pytest.raises(ValueError):
        oracle.solve_sherman(np.array([1.0, 1.0]), np.ones((3, 2)), np.ones((3, 2)))
    with pytest.raises(ValueError):
        oracle.solve_sherman(np.array([1.0, -1.0]), np.ones((2, 2)), np.ones((2, 2)))
    bad = np.ones((2, 2))
    bad[0, 0] = np.inf
    with pytest.raises(ValueError):
        oracle.solve_sherman(np.array([1.0, 1.0]), bad, np.ones((2, 2)))
    with pytest.raises(oracle.OracleSingularUpdate) as info:
        oracle.sweep_grouped(np.array([-1.0]), np.array([[1.0]]), np.array([[1.0]]))
    assert info.value.level == 1
