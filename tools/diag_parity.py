"""Per-block-family parity diagnostics of the CUDA path vs the golden reference outputs."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]

import oracle  # noqa: E402
from conftest import golden_names, load_golden  # noqa: E402
from paper_2512_02293_b200.device import DeviceProblem  # noqa: E402


def rel(a, b):
    s = np.abs(b).max(initial=0.0)
    return np.abs(a - b).max(initial=0.0) / s if s > 0 else np.abs(a).max(initial=0.0)


for name in golden_names():
    P, out, opts = load_golden(name)
    dp = DeviceProblem(P, opts)
    dp.linearize()
    H_pp, H_pd, H_dd, g_p, g_d = dp.export_normal_eq()
    L = oracle.Layout(P, opts)
    H_imu, g_imu = oracle.vi_ba._imu_part(P, L)
    dx, dxd = dp.solve_step(opts["damping"])
    # oracle step from the GPU's own linearisation (isolates solve error from linearisation error)
    dx2, dxd2 = oracle.solve_step_dense(L, opts, H_pp, H_pd, H_dd, g_p, g_d, opts["damping"])
    print(f"{name:18s} Hvis {rel(H_pp - H_imu, out['H_pp'] - H_imu):.1e} Himu {rel(H_pp, out['H_pp']):.1e} "
          f"gvis {rel(g_p - g_imu, out['g_p'] - g_imu):.1e} Hdd {rel(H_dd, out['H_dd']):.1e} "
          f"gd {rel(g_d, out['g_d']):.1e} Hpd {rel(H_pd, out['H_pd']):.1e} | dx {rel(dx, out['dx']):.1e} "
          f"dxd {rel(dxd, out['dxd']):.1e} | solve-only dx {rel(dx, dx2):.1e} dxd {rel(dxd, dxd2):.1e} "
          f"| lin-only dx {rel(dx2, out['dx']):.1e} dxd {rel(dxd2, out['dxd']):.1e}")
    dp.close()
