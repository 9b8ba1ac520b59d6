"""Host-side logic of the drop-in (no GPU): API surface, validation that
happens before any device work, sharding helpers, input generators, and the
reduced-coordinate algebra the kernels implement (checked with the numpy
model against the oracle)."""

import numpy as np
import pytest

import oracle
import reduced_model as M
import paper_1302_3876_b200 as P
from golden_io import ism_cases, rel_err
from paper_1302_3876_b200 import workloads as W


def test_public_names_match_reference_hot_path():
    for name in ("analysis_step", "solve_sherman", "solve_sherman_blocked", "solve_analysis",
                 "SolverResult", "SolverChoice", "SelectionOperator", "ObservationBatch",
                 "SingularUpdateError", "long_op_count", "member_deviations", "innovations",
                 "level_blocks", "GROUP_LEVELS", "SINGULAR_TOL"):
        assert hasattr(P, name), name
    assert P.SINGULAR_TOL == 1e-14 and issubclass(P.SingularUpdateError, ArithmeticError)
    e = P.SingularUpdateError(3, 1e-16)
    assert e.level == 3 and e.denominator == 1e-16


def test_long_op_count():
    assert P.long_op_count(3, 3) == 108 and P.long_op_count(1, 1) == 6
    assert P.long_op_count(4, 10) == 600
    with pytest.raises(ValueError):
        P.long_op_count(0, 5)


def test_level_blocks():
    blocks = P.level_blocks(nens=3, level=0, workers=2)
    assert blocks[0][0] == 0 and blocks[-1][1] == 6 and sum(b - a for a, b in blocks) == 6
    for level in range(1, 4):
        b = P.level_blocks(nens=3, level=level, workers=4)
        assert b[0][0] == level and b[-1][1] == 6
    with pytest.raises(ValueError):
        P.level_blocks(3, 4, 1)


def test_selection_operator_validation():
    with pytest.raises(ValueError):
        P.SelectionOperator.from_indices([])
    with pytest.raises(ValueError):
        P.SelectionOperator.from_indices([2, 1])
    with pytest.raises(ValueError):
        P.SelectionOperator.from_indices([-1, 3])
    h = P.SelectionOperator.from_indices([0, 3, 6])
    assert h.nobs(10) == 3 and P.SelectionOperator.identity().nobs(7) == 7
    x = np.arange(20.0).reshape(10, 2)
    assert np.array_equal(h.apply(x), x[[0, 3, 6]])
    ident = P.SelectionOperator.identity()
    assert ident.apply(x) is x
    with pytest.raises(IndexError):
        h.apply(np.ones((5, 2)))


def test_solver_choice_errors():
    with pytest.raises(ValueError):
        P.solve_analysis("bogus", np.ones(2), np.ones((2, 2)), np.ones((2, 2)))
    with pytest.raises(NotImplementedError):
        P.solve_analysis("cholesky", np.ones(2), np.ones((2, 2)), np.ones((2, 2)))
    with pytest.raises(ValueError):
        P.solve_sherman_blocked(np.ones(2), np.ones((2, 2)), np.ones((2, 2)), workers=0)


def test_analysis_step_argument_errors_before_device():
    h = P.SelectionOperator.from_indices([1, 4])
    obs = P.ObservationBatch(y=np.zeros(2), perturbed=np.zeros((2, 4)), perturbations=np.zeros((2, 4)))
    with pytest.raises(ValueError):
        P.analysis_step(np.ones((6, 1)), obs, h, np.ones(2))
    with pytest.raises(ValueError):
        P.analysis_step(np.ones(6), obs, h, np.ones(2))
    with pytest.raises(IndexError):
        P.analysis_step(np.ones((3, 4)), obs, h, np.ones(2))
    with pytest.raises(ValueError):
        P.analysis_step(np.ones((6, 4)), obs, h, np.array([1.0, -1.0]))
    with pytest.raises(ValueError):
        P.analysis_step(np.ones((6, 4)), obs, h, np.ones(3))
    with pytest.raises(ValueError):  # influence matrix shape (enkf.py:194-198), checked before the device
        P.analysis_step(np.ones((6, 4)), obs, h, np.ones(2), localization=np.ones((3, 3)))
    with pytest.raises(ValueError):
        P.analysis_step(np.ones((6, 4)), obs, h, np.ones(2),
                        localization=P.influence_matrix_cyclic(7, P.SelectionOperator.identity()))
    with pytest.raises(ValueError):
        P.analysis_step(np.ones((6, 4)), obs, h, np.ones(2), solver="nope")
    # an empty observation set (identity H on zero states): the reference raises
    # ValueError from its sweep's first rank-1 update (sherman.py:187)
    empty = P.ObservationBatch(y=np.zeros(0), perturbed=np.zeros((0, 4)), perturbations=np.zeros((0, 4)))
    with pytest.raises(ValueError):
        P.analysis_step(np.ones((0, 4)), empty, P.SelectionOperator.identity(), np.ones(0))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_rows_cover(world):
    ns = 1000
    shards = [W.shard_rows(ns, world, k) for k in range(world)]
    assert shards[0][0] == 0 and shards[-1][1] == ns
    assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
    idx = np.sort(np.random.default_rng(1).choice(ns, 300, replace=False))
    spans = [W.obs_slice(idx, lo, hi) for lo, hi in shards]
    assert spans[0][0] == 0 and spans[-1][1] == 300
    for (lo, hi), (a, b) in zip(shards, spans):
        assert np.all((idx[a:b] >= lo) & (idx[a:b] < hi))


def test_generators_deterministic_and_shaped():
    a, b = W.config4(10), W.config4(10)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.perturbed, b.perturbed)
    ns, nobs, n = a.shape
    assert (ns, nobs, n) == (1 << 14, 1 << 10, 128)
    assert np.all(np.diff(a.indices) > 0) and a.indices[-1] < ns
    assert a.r.min() >= 0.25 and a.r.max() <= 1.0
    p1 = W.config1()
    assert p1.shape == (40, 20, 20) and np.all(p1.r == 0.01)
    p3 = W.config3()
    assert p3.shape == (16641, 1089, 96)


def test_reduced_algebra_matches_oracle_solve():
    """The Gram-level Sherman-Morrison recursion (what ism_levels_kernel runs)
    reproduces the reference sweep's Z and A = V'Z."""
    for k, (_, r, v, d, z_ref, _, _) in enumerate(ism_cases()):
        z, a = M.solve(r, v, d)
        assert rel_err(z, z_ref) <= 1e-11, k


def test_reduced_algebra_matches_oracle_analysis():
    for p in (W.config1(), W.config3(), W.config4(10)):
        xa = M.analysis(p.x, p.perturbed, p.indices, p.r)
        assert rel_err(xa, oracle.analysis_step(p.x, p.perturbed, p.indices, p.r)) <= 1e-11


def test_reduced_levels_report_first_singular_level():
    g = np.zeros((3, 6))
    g[0, 0] = 0.5
    g[1, 1] = 2.0
    g[2, 2] = -1.0  # den_3 = 1 + (-1) = 0
    with pytest.raises(M.ModelSingular) as info:
        M.levels(g)
    assert info.value.level == 3
