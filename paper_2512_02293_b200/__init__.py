"""B200-native dense visual-inertial bundle adjustment (VIGS-SLAM VI-BA hot path).

Drop-in for ``vislam.solver.solve_vi_ba`` (/root/reference/pkg/src/vislam/solver.py:344):
the solve runs in hand-written sm_100a CUDA kernels behind the C-ABI declared in
``include/vba.h``; this package is the Python host layer mirroring the
reference interface.
"""

__version__ = "0.1.0"
