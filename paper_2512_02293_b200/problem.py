"""Packing a reference-style ``FrameGraph`` into flat arrays, and writing results back.

The packed problem is a dict of numpy arrays (fp64 unless noted):

  kid[K] (int64)  q[K,4] p[K,3] v[K,3] bg[K,3] ba[K,3] ts[K]
  doff[K+1] (int64)  pix[n_disp,2]  disp[n_disp]
  ei[E] ej[E] (int64, keyframe *indices*)  eoff[E+1] (int64 rows)
  epix[R,2] tgt[R,2] w[R,2]
  fi[F] fj[F] (int64)  f_dt[F] f_dR[F,4] f_dp[F,3] f_dv[F,3] f_Jr[F,3,3]
  f_Jp[F,3,6] f_Jv[F,3,6] f_cov[F,15,15] f_bhat[F,6]
  grav_q[4] grav_G  intr[4]=(fx,fy,cx,cy)  Tcb[7]=(q wxyz,t) has_Tcb

It is what the device uploader consumes and what the test oracle reads.  The
graph is read duck-typed, so objects from the reference package
(/root/reference/pkg/src/vislam/solver.py:37-79, residuals.py:34-137,
imu.py:29-74) and from ``paper_2512_02293_b200.types`` both work.

Validation mirrors where the reference raises ``ValueError``:
edge row count vs source disparities (residuals.py:181-183), positive
disparities (residuals.py:184-185), IMU dt vs state timestamps
(residuals.py:281-284).
"""

from __future__ import annotations

import numpy as np


def pack_graph(graph) -> dict:
    kfs = list(graph.keyframes)
    K = len(kfs)
    index = {kf.kid: n for n, kf in enumerate(kfs)}
    P: dict = {}
    P["kid"] = np.array([kf.kid for kf in kfs], dtype=np.int64)
    P["q"] = np.array([np.asarray(kf.state.pose.rotation.q, float) for kf in kfs]).reshape(K, 4)
    P["p"] = np.array([np.asarray(kf.state.pose.translation, float) for kf in kfs]).reshape(K, 3)
    P["v"] = np.array([np.asarray(kf.state.velocity, float) for kf in kfs]).reshape(K, 3)
    P["bg"] = np.array([np.asarray(kf.state.bias.gyro_bias, float) for kf in kfs]).reshape(K, 3)
    P["ba"] = np.array([np.asarray(kf.state.bias.accel_bias, float) for kf in kfs]).reshape(K, 3)
    P["ts"] = np.array([float(kf.state.timestamp) for kf in kfs], dtype=float)
    counts = np.array([len(kf.disparities) for kf in kfs], dtype=np.int64)
    P["doff"] = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    P["pix"] = (np.concatenate([np.asarray(kf.pixels, float).reshape(-1, 2) for kf in kfs])
                if K else np.zeros((0, 2)))
    P["disp"] = (np.concatenate([np.asarray(kf.disparities, float).reshape(-1) for kf in kfs])
                 if K else np.zeros(0))
    if len(P["disp"]) and P["disp"].min() <= 0.0:
        raise ValueError("disparities must be strictly positive")

    edges = list(graph.vision_edges)
    E = len(edges)
    P["ei"] = np.array([index[e.i] for e in edges], dtype=np.int64)
    P["ej"] = np.array([index[e.j] for e in edges], dtype=np.int64)
    rows = np.array([len(e.pixels) for e in edges], dtype=np.int64)
    for e, n, i in zip(edges, rows, P["ei"]):
        if n != counts[i]:
            raise ValueError("disparity length must match edge pixel list")
        if len(e.targets) != n or len(e.weights) != n:
            raise ValueError("pixels, targets and weights must have equal length")
    P["eoff"] = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    if E:
        P["epix"] = np.concatenate([np.asarray(e.pixels, float).reshape(-1, 2) for e in edges])
        P["tgt"] = np.concatenate([np.asarray(e.targets, float).reshape(-1, 2) for e in edges])
        P["w"] = np.concatenate([np.asarray(e.weights, float).reshape(-1, 2) for e in edges])
    else:
        P["epix"] = P["tgt"] = P["w"] = np.zeros((0, 2))
    if len(P["w"]) and np.any(P["w"] < 0.0):
        raise ValueError("weights must be non-negative")

    ies = list(graph.inertial_edges)
    F = len(ies)
    P["fi"] = np.array([index[i] for i, _, _ in ies], dtype=np.int64)
    P["fj"] = np.array([index[j] for _, j, _ in ies], dtype=np.int64)
    P["f_dt"] = np.array([float(d.dt_total) for _, _, d in ies], dtype=float)
    P["f_dR"] = np.array([np.asarray(d.delta_R.q, float) for _, _, d in ies]).reshape(F, 4)
    P["f_dp"] = np.array([np.asarray(d.delta_p, float) for _, _, d in ies]).reshape(F, 3)
    P["f_dv"] = np.array([np.asarray(d.delta_v, float) for _, _, d in ies]).reshape(F, 3)
    P["f_Jr"] = np.array([np.asarray(d.J_rot, float) for _, _, d in ies]).reshape(F, 3, 3)
    P["f_Jp"] = np.array([np.asarray(d.J_pos, float) for _, _, d in ies]).reshape(F, 3, 6)
    P["f_Jv"] = np.array([np.asarray(d.J_vel, float) for _, _, d in ies]).reshape(F, 3, 6)
    P["f_cov"] = np.array([np.asarray(d.covariance, float) for _, _, d in ies]).reshape(F, 15, 15)
    P["f_bhat"] = np.array([np.concatenate([d.bias_lin_point.gyro_bias, d.bias_lin_point.accel_bias])
                            for _, _, d in ies], dtype=float).reshape(F, 6)
    for f in range(F):
        dt = P["ts"][P["fj"][f]] - P["ts"][P["fi"][f]]
        if abs(dt - P["f_dt"][f]) > 1e-6:
            raise ValueError(f"delta spans {P['f_dt'][f]:.6f}s but states are {dt:.6f}s apart")

    P["grav_q"] = np.asarray(graph.gravity.R_wg.q, float).copy()
    P["grav_G"] = float(graph.gravity.magnitude)
    k = graph.intrinsics
    P["intr"] = np.array([k.fx, k.fy, k.cx, k.cy], dtype=float)
    T = getattr(graph, "T_cb", None)
    P["has_Tcb"] = T is not None
    P["Tcb"] = (np.concatenate([np.asarray(T.rotation.q, float), np.asarray(T.translation, float)])
                if T is not None else np.array([1.0, 0, 0, 0, 0, 0, 0]))
    return P


def options_dict(opts) -> dict:
    names = ("max_iterations", "damping", "damping_up", "damping_down", "rel_decrease_tol",
             "step_tol", "max_damping", "frozen_keyframes", "optimize_gravity",
             "optimize_velocity_bias", "use_schur", "ridge")
    return {n: getattr(opts, n) for n in names}


def _rotation_exact(cls, q):
    """A ``cls`` rotation holding exactly the solver's canonical quaternion.  The device already
    normalised it (qcanon, as Rotation.__init__ does, geometry.py:94-98); constructing through
    __init__ would renormalise and can move the last ulp (cf. frontend.py:565-573)."""
    r = cls.identity()
    r.q = np.asarray(q, dtype=float).reshape(4).copy()
    return r


def write_back(graph, q, p, v, bg, ba, disp, grav_q, opts) -> None:
    """Assign new state objects like solver.py:326-341 (_apply_step) does.

    Frozen keyframes keep their objects (bit-identical gauge, solver.py:165-170);
    disparity arrays are replaced for every keyframe (disparity columns are
    never frozen); gravity is replaced only when it was optimized.
    """
    frozen = set(opts.frozen_keyframes)
    doff = 0
    for n, kf in enumerate(graph.keyframes):
        nd = len(kf.disparities)
        if nd:
            kf.disparities = np.asarray(disp[doff:doff + nd], dtype=float).copy()
        doff += nd
        if kf.kid in frozen:
            continue
        st = kf.state
        rot = _rotation_exact(type(st.pose.rotation), q[n])
        pose = type(st.pose)(rot, np.asarray(p[n], float).copy())
        if opts.optimize_velocity_bias:
            bias = type(st.bias)(np.asarray(bg[n], float).copy(), np.asarray(ba[n], float).copy())
            vel = np.asarray(v[n], float).copy()
        else:
            bias, vel = st.bias, st.velocity
        kf.state = type(st)(pose, vel, bias, st.timestamp)
    if opts.optimize_gravity:
        g = graph.gravity
        graph.gravity = type(g)(_rotation_exact(type(g.R_wg), grav_q), g.magnitude)
