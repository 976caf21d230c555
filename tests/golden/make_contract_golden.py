"""Goldens for the reference's solver contract (pkg/tests/test_solver.py), run by the REFERENCE.

Each window of /root/reference/pkg/tests/test_solver.py is rebuilt here with the
reference's own fixtures (pkg/tests/windows.py build_window / perturb_graph and
the seeds test_solver.py uses), its per-pixel inputs rounded to fp32 (what the
B200 path stores), and solved by vislam.solver.solve_vi_ba with the test's
options.  The packed inputs, the reference's SolveReport and final states, the
ground-truth translations (for the ATE contract) and a dense-path solve where
the test compares Schur and dense steps are stored in
tests/golden/contract/<name>.npz for tests/test_gpu_dropin.py, which runs the
same contract through paper_2512_02293_b200.solver.solve_vi_ba on the GPU.

Run:  python tests/golden/make_contract_golden.py   (build container only)
"""

from __future__ import annotations

import copy
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "contract")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from make_golden import round_fp32  # noqa: E402
from vislam import solver as S  # noqa: E402
from vislam.geometry import Rotation  # noqa: E402
from vislam.residuals import GravityModel  # noqa: E402
from windows import build_window, perturb_graph  # noqa: E402

from paper_2512_02293_b200.problem import pack_graph  # noqa: E402

OPT_KEYS = ("max_iterations", "damping", "damping_up", "damping_down", "rel_decrease_tol", "step_tol",
            "max_damping", "frozen_keyframes", "optimize_gravity", "optimize_velocity_bias", "use_schur", "ridge")


def report_dict(rep):
    return dict(iterations=rep.iterations, initial_cost=rep.initial_cost, final_cost=rep.final_cost,
                cost_trajectory=list(rep.cost_trajectory), termination=rep.termination,
                condition_warnings=list(rep.condition_warnings))


def save(name, graph, opts, truth=None, dense=False, **extra):
    graph = round_fp32(graph)
    P = pack_graph(graph)
    out = {"in_" + k: np.asarray(v) for k, v in P.items()}
    out["energy"] = np.array(S.total_energy(graph))
    g = copy.deepcopy(graph)
    rep = S.solve_vi_ba(g, opts)
    F = pack_graph(g)
    for k in ("q", "p", "v", "bg", "ba", "disp", "grav_q"):
        out["final_" + k] = F[k]
    out["final_energy"] = np.array(S.total_energy(g))
    meta = dict(opts={k: getattr(opts, k) for k in OPT_KEYS}, report=report_dict(rep), **extra)
    if dense:
        gd = copy.deepcopy(graph)
        od = copy.deepcopy(opts)
        od.use_schur = False
        repd = S.solve_vi_ba(gd, od)
        Fd = pack_graph(gd)
        for k in ("q", "p", "v", "disp"):
            out["dense_" + k] = Fd[k]
        meta["dense_report"] = report_dict(repd)
    if truth is not None:
        out["truth_p"] = np.array([t.pose.translation for t in truth])
    out["meta"] = np.array(json.dumps(meta))
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {len(P['kid'])} kf, {len(P['ei'])} edges; {rep.iterations} it, {rep.termination}, "
          f"costs {rep.cost_trajectory[0]:.3e} -> {rep.final_cost:.3e} ({os.path.getsize(path) / 1e3:.0f} kB)")


def main():
    SO = S.SolveOptions
    rng = np.random.default_rng(23)                                  # test_solver.py:58-68
    g, _ = build_window(rng, n_kf=3, n_px=8)
    perturb_graph(g, rng)
    save("zero_iterations", g, SO(max_iterations=0))

    rng = np.random.default_rng(24)                                  # :71-77
    g, truth = build_window(rng, n_kf=8, n_px=30)
    perturb_graph(g, rng, rot_deg=2.0, trans_m=0.05)
    save("recovers_perturbed", g, SO(max_iterations=15), truth=truth)

    rng = np.random.default_rng(25)                                  # :80-87
    g, _ = build_window(rng, n_kf=5, n_px=15)
    perturb_graph(g, rng, rot_deg=3.0, trans_m=0.08)
    save("strictly_decreasing", g, SO(max_iterations=8))

    rng = np.random.default_rng(26)                                  # :90-103
    g, _ = build_window(rng, n_kf=5, n_px=10, vision_weight=0.0)
    perturb_graph(g, rng, rot_deg=1.0, trans_m=0.03, vel=0.05)
    save("zero_weight_vision", g, SO(max_iterations=25))

    for n_kf, n_px in ((3, 20), (5, 50), (4, 7)):                   # :106-121
        rng = np.random.default_rng(100 + n_kf * 10 + n_px)
        g, _ = build_window(rng, n_kf=n_kf, n_px=n_px)
        perturb_graph(g, rng, rot_deg=2.0, trans_m=0.05)
        save(f"schur_dense_{n_kf}_{n_px}", g, SO(max_iterations=3, use_schur=True), dense=True)

    rng = np.random.default_rng(27)                                  # :124-138
    g, _ = build_window(rng, n_kf=5, n_px=12)
    perturb_graph(g, rng)
    save("frozen_bit_identical", g, SO(max_iterations=5))

    rng = np.random.default_rng(28)                                  # :141-153
    g, _ = build_window(rng, n_kf=4, n_px=10)
    perturb_graph(g, rng)
    save("deterministic", g, SO(max_iterations=6))

    rng = np.random.default_rng(30)                                  # :165-175
    g, _ = build_window(rng, n_kf=5, n_px=15)
    g.gravity = GravityModel(g.gravity.R_wg * Rotation.exp(np.array([0.01, -0.02, 0.0])))
    save("gravity_optimization", g, SO(max_iterations=10, optimize_gravity=True))


if __name__ == "__main__":
    main()
