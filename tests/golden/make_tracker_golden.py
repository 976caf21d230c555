"""A real tracking window from the REFERENCE's tracker, for the device-window replay test.

Drives vislam's tracker (frontend.process_frame over the reference's synthetic figure-eight
dataset, 0.5 px correspondence noise, provider stride 40 -> 192 px per keyframe, an
8-keyframe window) past full initialisation and several evictions, serialises it with
TrackerState.to_dict (frontend.py:209-294; the JSON checkpoint format) into
tests/golden/tracker/window.json.gz, and records the reference's window solve on it
(_tracking_solve, frontend.py:435-450: SolveOptions(max_iterations=4, frozen first kid))
in tests/golden/tracker/window_solve.npz.  Build container only.
"""
import copy
import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from vislam.frontend import KeyframePolicy, make_tracker, process_frame  # noqa: E402
from vislam.initialization import InitConfig  # noqa: E402
from vislam.solver import SolveOptions, solve_vi_ba  # noqa: E402
from vislam.synth import SyntheticProvider, TrajectoryModel, make_dataset  # noqa: E402


def main():
    model = TrajectoryModel(family="figure8", amplitude=1.5, period=12.0, duration=12.0, yaw_policy="tangent")
    ds = make_dataset(model, sigma_px=0.5)
    prov = SyntheticProvider(ds, stride=40)
    tr = make_tracker(prov, policy=KeyframePolicy(window_size=8), init_cfg=InitConfig(n_vis_init=6, n_iner_init=10),
                      imu_period=1.0 / ds.imu_rate)
    for f in range(110):
        t = ds.frame_time(f)
        imu = [] if f == 0 else ds.imu_between(ds.frame_time(f - 1), t)
        process_frame(tr, f, t, imu)
    d = tr.to_dict()
    out = os.path.join(HERE, "tracker")
    os.makedirs(out, exist_ok=True)
    with gzip.open(os.path.join(out, "window.json.gz"), "wt") as fh:
        json.dump(d, fh)
    g = copy.deepcopy(tr.graph)
    frozen = (g.keyframes[0].kid,)
    rep = solve_vi_ba(g, SolveOptions(max_iterations=4, frozen_keyframes=frozen))
    np.savez_compressed(
        os.path.join(out, "window_solve.npz"),
        final_p=np.array([kf.state.pose.translation for kf in g.keyframes]),
        final_q=np.array([kf.state.pose.rotation.q for kf in g.keyframes]),
        final_v=np.array([kf.state.velocity for kf in g.keyframes]),
        final_disp=np.concatenate([kf.disparities for kf in g.keyframes]),
        report=np.array(json.dumps(dict(iterations=rep.iterations, initial_cost=rep.initial_cost,
                                        final_cost=rep.final_cost, cost_trajectory=list(rep.cost_trajectory),
                                        termination=rep.termination, condition_warnings=list(rep.condition_warnings)))),
        frozen=np.array(frozen))
    print(f"phase {tr.phase}, {len(g.keyframes)} kf, {len(g.vision_edges)} edges, "
          f"{len(g.inertial_edges)} imu; solve {rep.iterations} it {rep.termination} "
          f"{rep.cost_trajectory[0]:.6e} -> {rep.final_cost:.6e}; "
          f"json {os.path.getsize(os.path.join(out, 'window.json.gz')) / 1e3:.0f} kB")


if __name__ == "__main__":
    main()
