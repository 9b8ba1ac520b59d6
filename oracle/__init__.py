"""CPU oracle for the EnKF analysis step — TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference `enkfkit`
analysis path (arXiv 1302.3876, `/root/reference/pkg/src/enkfkit`). It is the
checker the parity tests compare the CUDA path against, and the CPU arm that
`bench.py --impl reference` / `cpu_baseline` time.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU legs may import it; the product
package `paper_1302_3876_b200` never does and has no CPU fallback.

Pinning: every function here was checked against golden vectors produced by
running the reference itself in the build container
(`tests/golden/make_golden.py` → `tests/golden/*.npz`, checked by
`tests/test_oracle_golden.py`).
"""

from .enkf_oracle import (  # noqa: F401
    GROUP_LEVELS,
    SINGULAR_TOL,
    OracleDivergence,
    OracleSingularUpdate,
    analysis_step,
    analysis_step_chunked,
    analysis_step_localized,
    apply_selection,
    cycle_l96,
    inflate,
    influence_matrix_cyclic,
    innovations,
    l96_advance,
    l96_rk4_step,
    l96_tendency,
    long_op_count,
    member_deviations,
    solve_sherman,
    sweep_grouped,
    sweep_levelwise,
    validate_system,
)
