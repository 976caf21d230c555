"""fp64 numpy restatement of stage-2 inertial-only initialisation — TEST INFRASTRUCTURE.

Restates /root/reference/pkg/src/vislam/initialization.py:121-231 (``_fd_velocities``,
``_inertial_only_cost``, ``init_inertial_only``) on the packed problem dict of
``problem.pack_graph`` with oracle.vi_ba.inertial_residual (residuals.py:274-354).
Returns (log_scale, gravity quaternion, bias[6], velocities[K,3], report dict).
The product package never imports this module.
"""

from __future__ import annotations

import numpy as np

from .vi_ba import GRAV_BASIS, inertial_residual, qcanon, qexp, qmul


def fd_velocities(P):
    """initialization.py:121-134"""
    n = len(P["kid"])
    v = np.zeros((n, 3))
    for k in range(n):
        a, b = max(0, k - 1), min(n - 1, k + 1)
        dt = P["ts"][b] - P["ts"][a]
        if dt <= 0.0:
            raise ValueError("keyframe timestamps must increase")
        v[k] = (P["p"][b] - P["p"][a]) / dt
    return v


def _cost(P, s, grav_q, bias, vel):
    """initialization.py:137-149"""
    n = len(P["kid"])
    es = float(np.exp(s))
    S = dict(q=P["q"], p=es * np.asarray(P["p"]), v=vel, bg=np.tile(bias[:3], (n, 1)), ba=np.tile(bias[3:], (n, 1)),
             grav_q=grav_q, grav_G=P["grav_G"], ts=P["ts"])
    outs = [inertial_residual(P, f, state=S) for f in range(len(P["fi"]))]
    return sum(float((o[0] ** 2).sum()) for o in outs), outs


def init_inertial_only(P, max_iterations=60, damping=1e-4):
    """initialization.py:152-231"""
    n = len(P["kid"])
    if n < 2 or len(P["fi"]) == 0:
        raise ValueError("need at least two keyframes with inertial edges")
    s = 0.0
    grav = np.array(P["grav_q"], float)
    bias = np.concatenate([P["bg"][0], P["ba"][0]]).astype(float)
    vel = fd_velocities(P)
    dim = 9 + 3 * n
    lam = damping
    cost, outs = _cost(P, s, grav, bias, vel)
    traj = [cost]
    term = "max_iterations"
    iters = 0
    for _ in range(max_iterations):
        es = float(np.exp(s))
        H = np.zeros((dim, dim))
        g = np.zeros(dim)
        for f, (r, Ji, Jj, Jg) in enumerate(outs):
            ki, kj = int(P["fi"][f]), int(P["fj"][f])
            J = np.zeros((15, dim))
            J[:, 0] = Ji[:, 3:6] @ (es * P["p"][ki]) + Jj[:, 3:6] @ (es * P["p"][kj])
            J[:, 1:3] = Jg @ GRAV_BASIS
            J[:, 3:9] = Ji[:, 9:15] + Jj[:, 9:15]
            J[:, 9 + 3 * ki:12 + 3 * ki] = Ji[:, 6:9]
            J[:, 9 + 3 * kj:12 + 3 * kj] = Jj[:, 6:9]
            H += J.T @ J
            g += J.T @ r
        accepted = False
        while lam <= 1e8:
            Hd = H + np.diag(np.diag(H)) * lam + 1e-10 * np.eye(dim)
            try:
                dx = np.linalg.solve(Hd, -g)
            except np.linalg.LinAlgError:
                break
            s_new = s + float(dx[0])
            g_new = qcanon(qmul(grav, qexp(GRAV_BASIS @ dx[1:3])))
            b_new = bias + dx[3:9]
            v_new = vel + dx[9:].reshape(n, 3)
            c_new, o_new = _cost(P, s_new, g_new, b_new, v_new)
            if c_new < cost:
                rel = (cost - c_new) / max(cost, 1e-30)
                s, grav, bias, vel, cost, outs = s_new, g_new, b_new, v_new, c_new, o_new
                traj.append(cost)
                lam = max(lam * 0.5, 1e-12)
                accepted = True
                iters += 1
                if rel < 1e-10:
                    term = "converged"
                break
            lam *= 10.0
        if not accepted:
            term = "no_decrease_at_max_damping"
            break
        if term == "converged":
            break
    rep = dict(iterations=iters, initial_cost=traj[0], final_cost=cost, cost_trajectory=traj, termination=term)
    return s, grav, bias, vel, rep
