"""Solver registry of the drop-in (reference solvers.py:26-31, 91-112).

Only the iterative Sherman-Morrison solver is on the B200 path.  The
Cholesky and SVD baselines are dense CPU comparison solvers in the reference
(solvers.py:34-88) and are deliberately not provided here: selecting them
raises NotImplementedError instead of silently running something else.
"""

from __future__ import annotations

from enum import Enum


class SolverChoice(str, Enum):
    """solvers.py:26-31 (same members and values)."""

    SHERMAN = "sherman"
    CHOLESKY = "cholesky"
    SVD = "svd"


def _require_sherman(choice) -> None:
    choice = SolverChoice(choice)  # unknown name -> ValueError, as in solvers.py:104
    if choice is not SolverChoice.SHERMAN:
        raise NotImplementedError(
            f"solver {choice.value!r} is a CPU comparison baseline of the reference; "
            "the B200 path implements only 'sherman'")


def solve_analysis(choice, r, v, d, workers: int = 1):
    """solvers.py:91-112 — dispatch; 'sherman' runs `solve_sherman` on the GPU
    (``workers`` > 1 maps to `solve_sherman_blocked`, whose GPU result is
    identical for every worker count)."""
    from .sherman import solve_sherman, solve_sherman_blocked

    _require_sherman(choice)
    if workers > 1:
        return solve_sherman_blocked(r, v, d, workers=workers)
    return solve_sherman(r, v, d)
