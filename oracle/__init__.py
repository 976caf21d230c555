"""CPU oracle for the dense VI-BA hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in fp64 numpy, the reference algorithm of
``vislam.solver.solve_vi_ba`` and its callees
(/root/reference/pkg/src/vislam/solver.py:118-411, residuals.py:172-354,
geometry.py:23-223).  It is the *checker* for the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` leg may import it;
* the product package ``paper_2512_02293_b200`` never imports it and has no
  CPU fallback.

Parity pin: the restatement is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports
/root/reference/pkg/src in the build container and writes
``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.
"""

from .vi_ba import (  # noqa: F401
    Layout,
    apply_step,
    inertial_residual,
    linearize_dense,
    linearize_sparse,
    solve_step_dense,
    solve_step_sparse,
    solve_vi_ba,
    total_energy,
    vision_residual,
)
