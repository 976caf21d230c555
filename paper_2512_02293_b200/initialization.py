"""Staged IMU initialisation with the GPU solves.

Mirrors vislam.initialization (/root/reference/pkg/src/vislam/initialization.py):

* ``init_inertial_only(graph, cfg)`` (stage 2, initialization.py:152-231) runs in libvba
  (``vba_init_inertial``, csrc/vba_init.cu + the inertial factor kernel of csrc/vba_imu.cu):
  damped Gauss-Newton over [log-scale, gravity (2), shared bias (6), velocities (3K)] with
  the vision poses frozen;
* ``init_vision`` (stage 1, :64-83) and ``init_joint`` (stage 3, :251-260) are the GPU
  ``solver.solve_vi_ba`` with the reference's options;
* ``align_gravity`` (:86-118), ``_fd_velocities`` (:121-134) and ``apply_initialization``
  (:234-248) are the reference's closed-form seeds and in-place write-back, restated on the
  host (a K-term mean and per-keyframe object updates: no solver arithmetic);
* ``run_full_initialization`` (:263-286) chains them.

The graph is read duck-typed (reference classes or paper_2512_02293_b200.types); results
use the caller's own classes where the graph provides them.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .types import InitConfig, InitResult, SolveOptions, SolveReport

_TERM = {0: "max_iterations", 1: "converged", 2: "no_decrease_at_max_damping"}


def _fd_velocities(graph):
    """initialization.py:121-134: central-difference velocity seeds."""
    states = [kf.state for kf in graph.keyframes]
    n = len(states)
    v = np.zeros((n, 3))
    for k in range(n):
        a, b = max(0, k - 1), min(n - 1, k + 1)
        dt = states[b].timestamp - states[a].timestamp
        if dt <= 0.0:
            raise ValueError("keyframe timestamps must increase")
        v[k] = (np.asarray(states[b].pose.translation) - np.asarray(states[a].pose.translation)) / dt
    return v


def _gravity_like(graph, q, magnitude):
    from .problem import _rotation_exact
    g = graph.gravity
    return type(g)(_rotation_exact(type(g.R_wg), q), magnitude)


def init_inertial_only(graph, cfg=None):
    """initialization.py:152-231 on the GPU."""
    import torch

    from .window import _imu_record
    cfg = cfg if cfg is not None else InitConfig()
    kfs = list(graph.keyframes)
    n = len(kfs)
    if n < 2 or not graph.inertial_edges:
        raise ValueError("need at least two keyframes with inertial edges")
    if not L.cuda_available():
        raise RuntimeError("paper_2512_02293_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    index = {kf.kid: k for k, kf in enumerate(kfs)}
    lib = L.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    q = np.array([np.asarray(kf.state.pose.rotation.q, float) for kf in kfs])
    p = np.array([np.asarray(kf.state.pose.translation, float) for kf in kfs])
    ts = np.array([float(kf.state.timestamp) for kf in kfs])
    v0 = _fd_velocities(graph)
    ies = list(graph.inertial_edges)
    fi = np.array([index[i] for i, _, _ in ies], dtype=np.int32)
    fj = np.array([index[j] for _, j, _ in ies], dtype=np.int32)
    recs = np.array([_imu_record(d) for _, _, d in ies])
    dts = ts[fj] - ts[fi]
    bad = np.nonzero(np.abs(dts - recs[:, 0]) > 1e-6)[0]
    if len(bad):
        f = int(bad[0])
        raise ValueError(f"delta spans {recs[f, 0]:.6f}s but states are {dts[f]:.6f}s apart")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).to(dev)  # noqa: E731
    d_q, d_p, d_v0, d_imu = t(q), t(p), t(v0), t(recs)
    v_out = torch.empty(3 * n, dtype=torch.float64, device=dev)
    P = L.VbaInitProblem()
    P.n_kf, P.n_imu = n, len(ies)
    P.q, P.p, P.v0, P.imu = d_q.data_ptr(), d_p.data_ptr(), d_v0.data_ptr(), d_imu.data_ptr()
    P.h_imu_i, P.h_imu_j = fi.ctypes.data, fj.ctypes.data
    g = graph.gravity
    for a in range(4):
        P.grav_q[a] = float(g.R_wg.q[a])
    P.grav_G = float(g.magnitude)
    b0 = kfs[0].state.bias
    for a in range(3):
        P.bias0[a] = float(b0.gyro_bias[a])
        P.bias0[3 + a] = float(b0.accel_bias[a])
    O = L.VbaInitOptions()
    O.max_iterations = int(cfg.max_iterations_inertial)
    O.damping = float(cfg.damping)
    R = L.VbaInitResult()
    cap = int(cfg.max_iterations_inertial) + 2
    traj = (C.c_double * cap)()
    st = torch.cuda.current_stream(dev)
    rc = lib.vba_init_inertial(C.byref(P), C.byref(O), C.c_void_p(st.cuda_stream), C.byref(R), traj, cap,
                               C.c_void_p(v_out.data_ptr()))
    if rc == L.VBA_E_COV:
        raise ValueError("non-PSD preintegration covariance")
    L.check(rc)
    report = SolveReport(R.iterations, R.initial_cost, R.final_cost, [traj[k] for k in range(min(R.n_costs, cap))],
                         _TERM[R.termination], [])
    bias = type(b0)(np.array(R.bias[0:3]), np.array(R.bias[3:6]))
    return InitResult(gravity=_gravity_like(graph, np.array(R.grav_q[:]), g.magnitude), log_scale=float(R.log_scale),
                      velocities=v_out.cpu().numpy().reshape(n, 3), bias=bias, reports={"inertial": report})


def _frame_graph_like(graph, inertial_edges):
    return type(graph)(keyframes=graph.keyframes, vision_edges=graph.vision_edges, inertial_edges=inertial_edges,
                       gravity=graph.gravity, intrinsics=graph.intrinsics, T_cb=getattr(graph, "T_cb", None))


def init_vision(graph, cfg=None):
    """initialization.py:64-83: vision-only BA of the window on the GPU (poses only)."""
    from .solver import solve_vi_ba
    cfg = cfg if cfg is not None else InitConfig()
    if not graph.keyframes:
        raise ValueError("cannot initialize an empty window")
    opts = SolveOptions(max_iterations=cfg.max_iterations_vision, damping=cfg.damping,
                        frozen_keyframes=(graph.keyframes[0].kid,), optimize_velocity_bias=False)
    return solve_vi_ba(_frame_graph_like(graph, []), opts)


def align_gravity(states, deltas, magnitude=9.81, gravity_cls=None):
    """initialization.py:86-118 (closed form, host): the mean velocity-change direction mapped to
    a yaw-free rotation of the inertial gravity axis."""
    from .types import GravityModel, Rotation
    if len(states) < 2 or len(deltas) != len(states) - 1:
        raise ValueError("need one preintegrated delta per consecutive pair")
    votes = []
    for k, delta in enumerate(deltas):
        s_i, s_j = states[k], states[k + 1]
        Ri = Rotation(np.asarray(s_i.pose.rotation.q, float)).matrix()
        votes.append((np.asarray(s_j.velocity) - np.asarray(s_i.velocity) - Ri @ np.asarray(delta.delta_v))
                     / delta.dt_total)
    g_mean = np.mean(votes, axis=0)
    norm = np.linalg.norm(g_mean)
    if norm < 1e-8:
        raise ValueError("gravity direction unobservable from these windows")
    direction = g_mean / norm
    e3 = np.array([0.0, 0.0, 1.0])
    c = float(np.clip(direction @ e3, -1.0, 1.0))
    axis = np.cross(e3, direction)
    s = np.linalg.norm(axis)
    if s < 1e-12:
        rotvec = np.zeros(3) if c > 0.0 else np.array([np.pi, 0.0, 0.0])
    else:
        rotvec = axis / s * np.arctan2(s, c)
    G, R = (gravity_cls or (GravityModel, Rotation))
    return G(R.exp(rotvec), magnitude)


def apply_initialization(graph, result):
    """initialization.py:234-248: positions * exp(s), disparities / exp(s), velocities, bias and
    gravity replaced (in place)."""
    es = result.scale()
    for k, kf in enumerate(graph.keyframes):
        st = kf.state
        pose = type(st.pose)(st.pose.rotation, es * np.asarray(st.pose.translation))
        kf.state = type(st)(pose, np.array(result.velocities[k], copy=True), result.bias.copy(), st.timestamp)
        kf.disparities = kf.disparities / es
    graph.gravity = result.gravity.copy()


def init_joint(graph, cfg=None):
    """initialization.py:251-260: full visual-inertial GPU solve with free gravity."""
    from .solver import solve_vi_ba
    cfg = cfg if cfg is not None else InitConfig()
    if not graph.keyframes:
        raise ValueError("cannot initialize an empty window")
    opts = SolveOptions(max_iterations=cfg.max_iterations_joint, damping=cfg.damping,
                        frozen_keyframes=(graph.keyframes[0].kid,), optimize_gravity=True)
    return solve_vi_ba(graph, opts)


def run_full_initialization(graph, cfg=None):
    """initialization.py:263-286: the three stages in sequence, mutating the window."""
    cfg = cfg if cfg is not None else InitConfig()
    vision_report = init_vision(graph, cfg)
    fd_vel = _fd_velocities(graph)
    seeds = [type(kf.state)(kf.state.pose, fd_vel[k], kf.state.bias, kf.state.timestamp)
             for k, kf in enumerate(graph.keyframes)]
    deltas = [d for _, _, d in graph.inertial_edges]
    g = graph.gravity
    graph.gravity = align_gravity(seeds, deltas, magnitude=g.magnitude,
                                  gravity_cls=(type(g), type(g.R_wg)))
    result = init_inertial_only(graph, cfg)
    apply_initialization(graph, result)
    joint_report = init_joint(graph, cfg)
    result.gravity = graph.gravity.copy()
    result.velocities = np.stack([np.asarray(kf.state.velocity) for kf in graph.keyframes])
    result.bias = graph.keyframes[-1].state.bias.copy()
    result.reports["vision"] = vision_report
    result.reports["joint"] = joint_report
    return result
