"""CPU ORACLE — test infrastructure only, never part of the product path.

A float64 NumPy restatement of the reference DASH optimizer step (``/root/reference/pkg/src/
blockshampoo``, cited file:line per function) used to check the B200 kernels.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import
it.  The product package ``paper_2602_02016_b200`` never imports, calls or links anything here.

Pinning: the restatement is checked against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports the read-only reference in the build container and stores
inputs/outputs in ``tests/golden/*.npz``; ``tests/test_oracle.py`` replays them), and directly
against the live reference when ``/root/reference`` is present.
"""
from .core import (  # noqa: F401
    IterationReport,
    OracleConfig,
    batched_clenshaw,
    batched_coupled_newton,
    batched_newton_db,
    block_seed,
    build_structure,
    chunk_bounds,
    cheb_coefficients,
    graft_scale,
    init_state,
    multi_power_iteration,
    partition_layout,
    random_spd,
    refresh,
    step,
    accumulate,
)
