"""Generate golden vectors by running the REFERENCE solver (build container only).

Imports the reference package read-only from /root/reference/pkg/src (and its
test fixtures ``windows.py`` from /root/reference/pkg/tests), builds seeded
windows, rounds every per-pixel input to fp32-representable values (the B200
path stores them as fp32), and records the reference's own outputs:

* ``total_energy``                       (solver.py:118-131)
* ``_linearize``  H_pp, H_pd, H_dd, g_p, g_d (solver.py:173-251)
* ``_solve_step`` dx_full, dx_d at λ=1e-4  (solver.py:265-308)
* ``solve_vi_ba`` final states + SolveReport (solver.py:344-411)

Run:  python tests/golden/make_golden.py      (writes tests/golden/*.npz)
The GPU box never runs this (no /root/reference there); tests read the npz.
"""

from __future__ import annotations

import copy
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from vislam import solver as ref_solver  # noqa: E402
from vislam.geometry import Pose, Rotation  # noqa: E402
from vislam.residuals import GravityModel  # noqa: E402
from windows import build_window, perturb_graph  # noqa: E402

from paper_2512_02293_b200.problem import pack_graph  # noqa: E402


def to_reference_graph(g):
    """Rebuild a paper_2512_02293_b200.types graph with the reference classes."""
    from vislam.imu import BiasState, PreintegratedDelta
    from vislam.residuals import Intrinsics, PoseState, VisionEdge

    R = lambda r: Rotation(np.array(r.q, copy=True))  # noqa: E731
    kfs = [ref_solver.Keyframe(kf.kid, PoseState(
        Pose(R(kf.state.pose.rotation), kf.state.pose.translation.copy()),
        kf.state.velocity.copy(),
        BiasState(kf.state.bias.gyro_bias.copy(), kf.state.bias.accel_bias.copy()),
        kf.state.timestamp), kf.pixels.copy(), kf.disparities.copy()) for kf in g.keyframes]
    edges = [VisionEdge(e.i, e.j, e.pixels.copy(), e.targets.copy(), e.weights.copy())
             for e in g.vision_edges]
    imu = [(i, j, PreintegratedDelta(d.dt_total, R(d.delta_R), d.delta_p.copy(), d.delta_v.copy(),
                                     d.J_rot.copy(), d.J_pos.copy(), d.J_vel.copy(),
                                     d.covariance.copy(),
                                     BiasState(d.bias_lin_point.gyro_bias.copy(),
                                               d.bias_lin_point.accel_bias.copy())))
           for i, j, d in g.inertial_edges]
    k = g.intrinsics
    return ref_solver.FrameGraph(kfs, edges, imu, GravityModel(R(g.gravity.R_wg), g.gravity.magnitude),
                                 Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height))


def round_fp32(graph):
    """Make every per-pixel input exactly fp32-representable (shared by kf and edges)."""
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    pix = {}
    for kf in graph.keyframes:
        kf.pixels = f32(kf.pixels)
        kf.disparities = f32(kf.disparities)
        pix[kf.kid] = kf.pixels
    for e in graph.vision_edges:
        same = e.pixels.shape == pix[e.i].shape
        e.pixels = pix[e.i] if same else f32(e.pixels)
        e.targets = f32(e.targets)
        e.weights = f32(e.weights)
    return graph


def ref_outputs(graph, opts, iters):
    layout = ref_solver._Layout(graph, opts)
    out = {}
    out["energy"] = np.array(ref_solver.total_energy(graph))
    H_pp, H_pd, H_dd, g_p, g_d = ref_solver._linearize(graph, layout)
    out.update(H_pp=H_pp, H_pd=H_pd, H_dd=H_dd, g_p=g_p, g_d=g_d)
    dx, dxd = ref_solver._solve_step(layout, H_pp, H_pd, H_dd, g_p, g_d, opts.damping, True)
    out.update(dx=dx, dxd=dxd)
    # conditioning floor: the reference's own step change when every flow target
    # moves by less than one fp32 ulp (what any fp32 evaluation of r introduces)
    rng = np.random.default_rng(7)
    cdx = cdxd = 0.0
    for _ in range(3):
        g3 = copy.deepcopy(graph)
        for e in g3.vision_edges:
            sp = np.spacing(np.abs(e.targets.astype(np.float32))).astype(np.float64)
            e.targets = e.targets + sp * rng.uniform(-1.0, 1.0, e.targets.shape)
        lin3 = ref_solver._linearize(g3, ref_solver._Layout(g3, opts))
        d3, dd3 = ref_solver._solve_step(layout, *lin3, opts.damping, True)
        cdx = max(cdx, float(np.abs(d3 - dx).max() / max(np.abs(dx).max(), 1e-300)))
        if len(dxd) and np.abs(dxd).max() > 0:
            cdxd = max(cdxd, float(np.abs(dd3 - dxd).max() / np.abs(dxd).max()))
    out.update(cond_dx=np.array(cdx), cond_dxd=np.array(cdxd))
    g2 = copy.deepcopy(graph)
    o2 = copy.deepcopy(opts)
    o2.max_iterations = iters
    rep = ref_solver.solve_vi_ba(g2, o2)
    Pf = pack_graph(g2)
    for k in ("q", "p", "v", "bg", "ba", "disp", "grav_q"):
        out["final_" + k] = Pf[k]
    out["report"] = np.array(json.dumps(dict(
        iterations=rep.iterations, initial_cost=rep.initial_cost, final_cost=rep.final_cost,
        cost_trajectory=list(rep.cost_trajectory), termination=rep.termination,
        condition_warnings=list(rep.condition_warnings))))
    return out


def save(name, graph, opts, iters):
    graph = round_fp32(graph)
    P = pack_graph(graph)
    out = ref_outputs(graph, opts, iters)
    arrays = {"in_" + k: np.asarray(v) for k, v in P.items()}
    arrays.update({"out_" + k: np.asarray(v) for k, v in out.items()})
    arrays["opts"] = np.array(json.dumps({k: getattr(opts, k) for k in (
        "max_iterations", "damping", "damping_up", "damping_down", "rel_decrease_tol",
        "step_tol", "max_damping", "frozen_keyframes", "optimize_gravity",
        "optimize_velocity_bias", "use_schur", "ridge")} | {"max_iterations": iters}))
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: E={len(P['ei'])} K={len(P['kid'])} rows={len(P['tgt'])} "
          f"energy={float(out['energy']):.6e} -> {os.path.getsize(path)/1e3:.0f} kB")


def main():
    S = ref_solver.SolveOptions
    # 1) the reference's own recovery window (test_solver.py:71-77)
    rng = np.random.default_rng(24)
    g, _ = build_window(rng, n_kf=8, n_px=30)
    perturb_graph(g, rng, rot_deg=2.0, trans_m=0.05)
    save("win8_px30", g, S(), 6)

    # 2) gravity optimisation (test_solver.py:165-175)
    rng = np.random.default_rng(30)
    g, _ = build_window(rng, n_kf=5, n_px=15)
    g.gravity = GravityModel(g.gravity.R_wg * Rotation.exp(np.array([0.01, -0.02, 0.0])))
    perturb_graph(g, rng, rot_deg=1.0, trans_m=0.02)
    save("win5_gravity", g, S(optimize_gravity=True), 6)

    # 3) vision-only, pose-only states (init_vision path, initialization.py:64-83)
    rng = np.random.default_rng(41)
    g, _ = build_window(rng, n_kf=4, n_px=20)
    g = ref_solver.FrameGraph(g.keyframes, g.vision_edges, [], g.gravity, g.intrinsics)
    perturb_graph(g, rng)
    save("win4_sdof6", g, S(optimize_velocity_bias=False), 5)

    # 4) non-identity camera extrinsic
    rng = np.random.default_rng(42)
    g, _ = build_window(rng, n_kf=4, n_px=12)
    g.T_cb = Pose(Rotation.exp(np.array([0.02, -0.01, 0.03])), np.array([0.05, -0.02, 0.01]))
    perturb_graph(g, rng)
    save("win4_tcb", g, S(), 4)

    # 5) zero-weight vision, IMU-only convergence (test_solver.py:90-103)
    rng = np.random.default_rng(26)
    g, _ = build_window(rng, n_kf=5, n_px=10, vision_weight=0.0)
    perturb_graph(g, rng, rot_deg=1.0, trans_m=0.03, vel=0.05)
    save("win5_zero_vision", g, S(), 6)

    # 6) two frozen keyframes, longer edge span
    rng = np.random.default_rng(43)
    g, _ = build_window(rng, n_kf=6, n_px=16, edge_span=3)
    perturb_graph(g, rng, skip_frozen=(0, 3))
    save("win6_frozen2", g, S(frozen_keyframes=(0, 3)), 4)

    # 7) BASELINE config-0 shapes (reduced grid) from the bench generator
    from paper_2512_02293_b200.workloads import make_workload
    g = to_reference_graph(make_workload(0, grid=(12, 16)))
    save("cfg0_grid12x16", g, S(), 2)


if __name__ == "__main__":
    main()
