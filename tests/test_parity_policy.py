"""CPU checks of the full-size parity machinery (tests/parity_policy.py): the
oracle's two sweep routes and the long-double Woodbury truth agree with a dense
solve of (R + V V') Z = D on small systems, and the policy's pass rule."""

import numpy as np

import parity_policy as PP
from paper_1302_3876_b200 import workloads as W


def _dense_a(xo, y, r):
    n = xo.shape[1]
    v = (xo - xo.mean(axis=1, keepdims=True)) / np.sqrt(n - 1.0)
    d = y - xo
    return v.T @ np.linalg.solve(np.diag(r) + v @ v.T, d)


def test_routes_and_truth_match_dense_solve():
    g = np.random.Generator(np.random.Philox(77))
    nobs, n = 400, 24
    xo = g.standard_normal((nobs, 1)) + g.uniform(0.5, 2.0, (nobs, 1)) * g.standard_normal((nobs, n))
    r = g.uniform(0.25, 1.0, nobs)
    y = xo.mean(axis=1, keepdims=True) + np.sqrt(r)[:, None] * g.standard_normal((nobs, n))
    ref = _dense_a(xo, y, r)
    a = PP.obs_side_oracle(xo, y, r)
    scale = np.abs(ref).max()
    for route in ("grouped", "levelwise"):
        assert np.abs(a[route] - ref).max() <= 1e-11 * scale, route
    assert np.abs(PP.truth_a(xo, y, r, rows_per_chunk=64) - ref).max() <= 1e-12 * scale


def test_truth_is_closer_than_the_oracle_at_scale():
    """At 2^14 observations (config-4 distributions) the oracle's V'Z already
    carries cancellation error; the Woodbury truth agrees with an fp64 Woodbury
    solve far more tightly than the oracle's two routes agree with each other."""
    p = W.config4(6)
    xo = p.x[p.indices]
    a = PP.obs_side_oracle(xo, p.perturbed, p.r)
    a_w = PP.truth_a(xo, p.perturbed, p.r)
    n = xo.shape[1]
    v = (xo - xo.mean(axis=1, keepdims=True)) / np.sqrt(n - 1.0)
    w = v / p.r[:, None]
    a64 = np.linalg.solve(np.eye(n) + w.T @ v, w.T @ (p.perturbed - xo))
    scale = np.abs(a_w).max()
    spread = np.abs(a["grouped"] - a["levelwise"]).max() / scale
    assert np.abs(a64 - a_w).max() / scale <= 1e-13
    assert spread > 10 * np.abs(a64 - a_w).max() / scale


def test_policy_rule():
    assert PP.verdict(4, 9e-10)[0] and not PP.verdict(4, 2e-9)[0]
    # config 5: the bound widens to twice the measured oracle floor ...
    ok, bound = PP.verdict(5, 5e-9, floor=4e-9, err_vs_truth=1e-12)
    assert ok and bound == 8e-9
    # ... but never below 1e-9, and the truth error stays bounded by 1e-9
    assert PP.verdict(5, 9e-10, floor=1e-12, err_vs_truth=1e-12)[0]
    assert not PP.verdict(5, 5e-9, floor=4e-9, err_vs_truth=2e-9)[0]
    assert not PP.verdict(5, 9e-9, floor=4e-9, err_vs_truth=1e-12)[0]
