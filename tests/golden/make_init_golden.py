"""Goldens for stage-2 inertial-only initialisation, produced by the REFERENCE.

The windows of /root/reference/pkg/tests/test_initialization.py:150-235 (its fixtures and
seeds) are built with windows.build_window, solved by vislam.initialization, and stored in
tests/golden/init/<name>.npz (packed inputs, InitResult fields, the stage-2 report):

* doubled_scale  (:151-156)  positions halved, log-scale -> log 2
* gyro_bias      (:158-164)  injected bias, bias_hat = 0
* metric         (:166-170)  metric input, log-scale ~ 0
* equivariance_a / _b (:172-181)  the same window at scale 1 and 1.7
* full_pipeline  (:210-227)  run_full_initialization (all three stages)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from make_golden import round_fp32  # noqa: E402
from vislam.geometry import Pose, Rotation  # noqa: E402
from vislam.imu import BiasState  # noqa: E402
from vislam.initialization import init_inertial_only, run_full_initialization  # noqa: E402
from vislam.residuals import GravityModel, PoseState  # noqa: E402
from windows import build_window, perturb_graph  # noqa: E402

from paper_2512_02293_b200.problem import pack_graph  # noqa: E402

OUT = os.path.join(HERE, "init")


def rescale(graph, k):
    for kf in graph.keyframes:
        st = kf.state
        kf.state = PoseState(Pose(st.pose.rotation, k * st.pose.translation), k * st.velocity, st.bias.copy(),
                             st.timestamp)
        kf.disparities = kf.disparities / k


def save(name, graph, full=False):
    graph = round_fp32(graph)
    P = pack_graph(graph)
    out = {"in_" + k: np.asarray(v) for k, v in P.items()}
    res = run_full_initialization(graph) if full else init_inertial_only(graph)
    out.update(log_scale=np.array(res.log_scale), grav_q=np.asarray(res.gravity.R_wg.q), bias=res.bias.vector(),
               velocities=np.asarray(res.velocities))
    reps = {k: dict(iterations=r.iterations, initial_cost=r.initial_cost, final_cost=r.final_cost,
                    cost_trajectory=list(r.cost_trajectory), termination=r.termination)
            for k, r in res.reports.items() if hasattr(r, "iterations")}
    if full:
        F = pack_graph(graph)
        for k in ("q", "p", "v", "bg", "ba", "disp", "grav_q"):
            out["final_" + k] = F[k]
    out["meta"] = np.array(json.dumps(dict(reports=reps, full=full)))
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, f"scale {np.exp(res.log_scale):.6f}", {k: (v["iterations"], v["termination"]) for k, v in reps.items()})


def main():
    rng = np.random.default_rng(6)
    g, _ = build_window(rng, n_kf=8)
    rescale(g, 0.5)
    save("doubled_scale", g)
    rng = np.random.default_rng(7)
    tb = BiasState([0.01, -0.02, 0.005], [0.03, -0.01, 0.02])
    g, _ = build_window(rng, n_kf=8, bias=tb, bias_hat=BiasState())
    save("gyro_bias", g)
    rng = np.random.default_rng(8)
    g, _ = build_window(rng, n_kf=8)
    save("metric", g)
    rng = np.random.default_rng(9)
    g, _ = build_window(rng, n_kf=6)
    save("equivariance_a", g)
    rng = np.random.default_rng(9)
    g, _ = build_window(rng, n_kf=6)
    rescale(g, 1.7)
    save("equivariance_b", g)
    rng = np.random.default_rng(13)
    tb = BiasState([0.008, -0.012, 0.004], [0.02, 0.01, -0.015])
    gravity = GravityModel(Rotation.exp([0.06, -0.09, 0.0]))
    g, truth = build_window(rng, n_kf=10, gravity=gravity, bias=tb, bias_hat=BiasState())
    rescale(g, 0.5)
    perturb_graph(g, rng, rot_deg=0.3, trans_m=0.01, vel=0.01)
    save("full_pipeline", g, full=True)


if __name__ == "__main__":
    main()
