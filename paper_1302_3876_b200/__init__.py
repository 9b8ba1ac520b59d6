"""B200-native EnKF analysis step (iterative Sherman-Morrison, arXiv 1302.3876).

Drop-in for the hot path of the reference package `enkfkit`: the names below
keep the reference's signatures and semantics (reference __init__.py:11-84),
while the arithmetic runs in hand-written sm_100a CUDA (libenkf_b200.so,
C ABI in include/enkf_b200.h).  Out-of-scope reference components (models,
twin-experiment harness, Cholesky/SVD baselines, CLI) are not provided;
the Lorenz-96 forecast and a device-resident cycled driver are (lorenz96.py);
localized analysis (enkf.py:193-199) runs on the GPU, with the cyclic
influence matrix evaluated on the fly.
"""

from .enkf import (
    CyclicInfluence,
    ObservationBatch,
    SelectionOperator,
    analysis_step,
    inflate,
    influence_matrix_cyclic,
    innovations,
    member_deviations,
)
from .errors import (
    ConfigError,
    DivergenceError,
    NotPositiveDefiniteError,
    NumericalFailureError,
    SingularUpdateError,
)
from .sherman import (
    GROUP_LEVELS,
    SINGULAR_TOL,
    SolverResult,
    level_blocks,
    long_op_count,
    solve_sherman,
    solve_sherman_blocked,
)
from .lorenz96 import CycleResult, Lorenz96, Lorenz96Config, cycle_l96, forecast_step
from .solvers import SolverChoice, solve_analysis

__version__ = "0.1.0"

__all__ = [
    "ConfigError",
    "CycleResult",
    "CyclicInfluence",
    "DivergenceError",
    "GROUP_LEVELS",
    "Lorenz96",
    "Lorenz96Config",
    "NotPositiveDefiniteError",
    "NumericalFailureError",
    "ObservationBatch",
    "SINGULAR_TOL",
    "SelectionOperator",
    "SingularUpdateError",
    "SolverChoice",
    "SolverResult",
    "analysis_step",
    "cycle_l96",
    "forecast_step",
    "inflate",
    "influence_matrix_cyclic",
    "innovations",
    "level_blocks",
    "long_op_count",
    "member_deviations",
    "solve_analysis",
    "solve_sherman",
    "solve_sherman_blocked",
]
