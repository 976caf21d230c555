"""Goldens for the Sim(3) pose-graph BA, produced by the REFERENCE (build container only).

Runs vislam.loopclosure (imported read-only from /root/reference/pkg/src) on:

* ``circle_rel``  -- test_loopclosure.py:458-477: 61-node drifting circle, one exact loop
  (information 1e6 I), chain only, 30 iterations;
* ``exact``       -- :407-431: an exactly consistent 61-node graph (energy 0, untouched);
* ``vision_loop`` -- :510-540: 6 nodes from the reference's synthetic provider (stride 40),
  one dense vision loop edge (its two-view alignment from align_loop_pair), 15 iterations;
* ``vision_tcb``  -- the same window with a non-identity camera extrinsic and 1 px flow noise;
* ``stress``      -- paper_2512_02293_b200.workloads.make_pgba_workload(): 256 nodes, 8 loops
  of 48x64 correspondences (converted to the reference's classes, then stored).

Stored: the packed inputs (small graphs), the energy, the dense linearisation
(_linearize_pg: H_pp, H_pd sampled columns, H_dd, g_p, g_d), the damped Schur step at
lambda = damping (solver._solve_step through loopclosure's layout), and solve_pgba's
SolveReport plus final states -> tests/golden/pgba/<name>.npz.
Per-pixel inputs are rounded to fp32 first (what the GPU stores).
"""

from __future__ import annotations

import copy
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "pgba")
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from conftest import packed_hash  # noqa: E402

import vislam.loopclosure as LC  # noqa: E402
from vislam.geometry import Pose, Rotation, SimTransform  # noqa: E402
from vislam.residuals import Intrinsics, RelativePoseEdge, VisionEdge  # noqa: E402
from vislam.solver import SolveOptions, _solve_step  # noqa: E402

from paper_2512_02293_b200.pgba import pack_pose_graph  # noqa: E402

f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
CHAIN_INFO = np.diag([4e4] * 3 + [1e4] * 3 + [100.0])


def chain_from(states, info=None):
    info = CHAIN_INFO if info is None else info
    return [RelativePoseEdge(k, k + 1, states[k + 1] * states[k].inverse(), info) for k in range(len(states) - 1)]


def int_state(t):
    return SimTransform(Rotation.identity(), np.array(t, float), 1.0)


def round_fp32(g):
    for n in g.nodes:
        if n.pixels is not None:
            n.pixels = f32(n.pixels)
            n.disparities = f32(n.disparities)
    for lp in g.loops:
        if lp.vision is not None:
            v = lp.vision
            lp.vision = VisionEdge(v.i, v.j, g.node(v.i).pixels, f32(v.targets), f32(v.weights))
    return g


def to_reference(g):
    """paper_2512_02293_b200.types PoseGraph -> the reference's classes."""
    S = lambda s: SimTransform(Rotation(np.array(s.rotation.q)), s.translation.copy(), s.scale)  # noqa: E731
    nodes = [LC.PoseGraphNode(n.kid, S(n.state), None if n.pixels is None else n.pixels.copy(),
                              None if n.disparities is None else n.disparities.copy(), n.timestamp)
             for n in g.nodes]
    R = lambda e: RelativePoseEdge(e.i, e.j, S(e.measurement), e.information.copy())  # noqa: E731
    loops = [LC.LoopEdge(lp.i, lp.j, R(lp.relative), None if lp.vision is None else VisionEdge(
        lp.vision.i, lp.vision.j, lp.vision.pixels.copy(), lp.vision.targets.copy(), lp.vision.weights.copy()))
        for lp in g.loops]
    k = g.intrinsics
    return LC.PoseGraph(nodes, [R(e) for e in g.chain], loops, Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height),
                        None, g.min_loop_gap)


def save(name, graph, opts, store_inputs=True, extra=None):
    graph = round_fp32(graph)
    P = pack_pose_graph(graph)
    out = {}
    if store_inputs:
        out.update({"in_" + k: np.asarray(v) for k, v in P.items()})
    lay = LC._PgLayout(graph, opts)
    out["energy"] = np.array(LC.total_pg_energy(graph))
    H_pp, H_pd, H_dd, g_p, g_d = LC._linearize_pg(graph, lay)
    out.update(H_pp=H_pp, H_dd=H_dd, g_p=g_p, g_d=g_d)
    if H_pd.shape[1]:
        rng = np.random.default_rng(5)
        cols = np.sort(rng.choice(H_pd.shape[1], min(512, H_pd.shape[1]), replace=False))
        out["H_pd_cols"] = cols.astype(np.int64)
        out["H_pd"] = H_pd[:, cols]
        out["H_pd_maxabs"] = np.array(np.abs(H_pd).max())
    dx, dxd = _solve_step(lay, H_pp, H_pd, H_dd, g_p, g_d, opts.damping, True)
    out.update(dx=dx, dxd=dxd)
    g2 = copy.deepcopy(graph)
    rep, corr = LC.solve_pgba(g2, opts)
    F = pack_pose_graph(g2)
    for k in ("sq", "st", "ss", "disp"):
        out["final_" + k] = F[k]
    meta = dict(opts={k: getattr(opts, k) for k in (
        "max_iterations", "damping", "damping_up", "damping_down", "rel_decrease_tol", "step_tol", "max_damping",
        "frozen_keyframes", "optimize_gravity", "optimize_velocity_bias", "use_schur", "ridge")},
        report=dict(iterations=rep.iterations, initial_cost=rep.initial_cost, final_cost=rep.final_cost,
                    cost_trajectory=list(rep.cost_trajectory), termination=rep.termination,
                    condition_warnings=list(rep.condition_warnings)),
        input_hash=packed_hash(P), **(extra or {}))
    out["meta"] = np.array(json.dumps(meta))
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {len(P['kid'])} nodes, {len(P['vi'])} vision loops, {len(P['ri'])} relative edges; "
          f"{rep.iterations} it {rep.termination}, cost {rep.initial_cost:.4e} -> {rep.final_cost:.4e} "
          f"({os.path.getsize(path) / 1e3:.0f} kB)")


def drifting_circle(n=61, cumulative_scale=1.05):
    """test_loopclosure.py:382-397"""
    ang = np.linspace(0.0, 1.5 * np.pi, n)
    gt = [SimTransform(Rotation.exp(np.array([0, 0, a + np.pi / 2])),
                       np.array([2 * np.cos(a), 2 * np.sin(a), 0.1 * np.sin(3 * a)]), 1.0) for a in ang]
    sigma = cumulative_scale ** (1.0 / (n - 1))
    drift = [gt[0].copy()]
    for k in range(n - 1):
        rel = gt[k + 1] * gt[k].inverse()
        drift.append(SimTransform(Rotation(rel.rotation.q.copy()), rel.translation.copy(), sigma) * drift[k])
    return gt, drift


def main():
    gt, drift = drifting_circle()
    nodes = [LC.PoseGraphNode(k, drift[k].copy(), timestamp=float(k)) for k in range(61)]
    loop = LC.LoopEdge(0, 60, RelativePoseEdge(0, 60, gt[60] * gt[0].inverse(), np.eye(7) * 1e6))
    save("circle_rel", LC.PoseGraph(nodes, chain_from(drift), [loop]), SolveOptions(max_iterations=30))

    states = [int_state([k, 2.0 * k % 7, -(k % 3)]) for k in range(61)]
    nodes = [LC.PoseGraphNode(k, s.copy(), timestamp=float(k)) for k, s in enumerate(states)]
    loop = LC.LoopEdge(0, 60, RelativePoseEdge(0, 60, states[60] * states[0].inverse(), np.eye(7) * 1e6))
    save("exact", LC.PoseGraph(nodes, chain_from(states), [loop]), SolveOptions())

    from vislam.synth import SyntheticProvider, TrajectoryModel, make_dataset
    model = TrajectoryModel(family="figure8", amplitude=1.5, period=12.0, duration=12.0, yaw_policy="tangent")
    ds = make_dataset(model, sigma_px=0.0)
    prov = SyntheticProvider(ds, stride=40)
    grid, k = prov.grid_pixels(), prov.intrinsics()
    frames = [0, 2, 4, 6, 8, 10]
    gtv = [SimTransform.from_pose(ds.frame_pose(f)) for f in frames]
    drifted = [gtv[0].copy()]
    for n in range(1, 6):
        a = n / 5.0
        D = SimTransform(Rotation.exp(a * np.array([0.0, 0.0, 0.04])), a * np.array([0.12, -0.08, 0.05]), 1.0)
        drifted.append(D * gtv[n])
    raw = prov.edge(frames[0], frames[-1])
    vis = VisionEdge(0, 5, raw.pixels, raw.targets, raw.weights)
    d0 = 1.0 / prov.depth_hint(frames[0], grid)
    rel = LC.align_loop_pair(vis, d0, drifted[0], drifted[5], k)
    nodes = [LC.PoseGraphNode(n, drifted[n].copy(), pixels=grid if n == 0 else None,
                              disparities=d0.copy() if n == 0 else None, timestamp=float(n)) for n in range(6)]
    g = LC.PoseGraph(nodes, chain_from(drifted), [LC.LoopEdge(0, 5, rel, vis)], intrinsics=k, min_loop_gap=5)
    save("vision_loop", g, SolveOptions(max_iterations=15))

    rng = np.random.default_rng(11)
    T_cb = Pose(Rotation.exp(np.array([0.02, -0.03, 0.05])), np.array([0.05, -0.02, 0.01]))
    tg = raw.targets + rng.normal(0.0, 1.0, raw.targets.shape)
    vis2 = VisionEdge(0, 5, raw.pixels, tg, raw.weights * rng.uniform(0.2, 1.0, raw.weights.shape))
    nodes = [LC.PoseGraphNode(n, drifted[n].copy(), pixels=grid if n == 0 else None,
                              disparities=(d0 * rng.uniform(0.95, 1.05, d0.shape)) if n == 0 else None,
                              timestamp=float(n)) for n in range(6)]
    g = LC.PoseGraph(nodes, chain_from(drifted), [LC.LoopEdge(0, 5, rel, vis2)], intrinsics=k, T_cb=T_cb,
                     min_loop_gap=5)
    save("vision_tcb", g, SolveOptions(max_iterations=10))

    from paper_2512_02293_b200.workloads import make_pgba_workload
    g, _ = make_pgba_workload()
    save("stress", to_reference(g), SolveOptions(max_iterations=6),
         extra=dict(generator="make_pgba_workload()"))


if __name__ == "__main__":
    main()
