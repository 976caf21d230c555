"""fp64 numpy restatement of the reference's Sim(3) pose-graph BA (PGBA) — TEST INFRASTRUCTURE.

Restates, citing lines (paths relative to /root/reference/pkg/src/vislam/):

* Sim(3) maps: ``_sim3_w_matrix`` geometry.py:230-263, ``SimTransform`` compose /
  inverse / exp / log / retract / adjoint geometry.py:266-341, ``sim3_ad``
  geometry.py:344-354, ``sim3_right_jacobian_inv`` geometry.py:357-370 (scipy expm,
  as the reference);
* ``sim3_vision_residual`` loopclosure.py:225-307, ``relative_pose_residual``
  residuals.py:364-380;
* ``total_pg_energy`` loopclosure.py:378-390, ``_PgLayout`` :392-422,
  ``_linearize_pg`` :425-475, ``_pg_apply`` :489-499, ``solve_pgba`` :502-574
  (the damped Schur step is the VI-BA one, oracle.vi_ba.solve_step_dense =
  solver._solve_step, shared exactly as loopclosure.py:27,534 shares it).

Input is the packed pose-graph dict of ``paper_2512_02293_b200.pgba.pack_pose_graph``:

  kid[K] sq[K,4] st[K,3] ss[K] ts[K]            Sim(3) node states (sorted by kid)
  doff[K+1] pix[n_disp,2] disp[n_disp]           disparity variables (vision-loop sources only)
  vi[V] vj[V] veoff[V+1] vpix vtgt vw            vision loop edges (node indices, rows of the source)
  ri[R] rj[R] rq[R,4] rt[R,3] rs[R] rinfo[R,7,7] relative edges (loops without vision, then chain)
  intr[4] Tcb[7] has_Tcb n_loops

The product package never imports this module.
"""

from __future__ import annotations

import copy

import numpy as np
from scipy.linalg import expm

from .vi_ba import DISPARITY_FLOOR, _T_bc, hat, qcanon, qexp, qlog, qmat, qmul, solve_step_dense

SIM3_DOF = 7


# ----------------------------------------------------------------------------
# Sim(3)  (geometry.py:230-370); a state is (q wxyz, t, s)
# ----------------------------------------------------------------------------

def sim3_w(omega, sigma):
    """geometry.py:230-263"""
    theta = np.linalg.norm(omega)
    K = hat(omega)
    K2 = K @ K
    s = np.exp(sigma)
    eps = 1e-6
    if abs(sigma) < eps:
        C = 1.0
        if theta < eps:
            A, B = 0.5, 1.0 / 6.0
        else:
            t2 = theta * theta
            A = (1.0 - np.cos(theta)) / t2
            B = (theta - np.sin(theta)) / (t2 * theta)
    else:
        C = (s - 1.0) / sigma
        if theta < eps:
            s2 = sigma * sigma
            A = ((sigma - 1.0) * s + 1.0) / s2
            B = (s * (0.5 * s2 - sigma + 1.0) - 1.0) / (s2 * sigma)
        else:
            t2 = theta * theta
            d = sigma * sigma + t2
            A = (s * sigma * np.sin(theta) + theta * (1.0 - s * np.cos(theta))) / (theta * d)
            B = (C - ((s * np.cos(theta) - 1.0) * sigma + s * np.sin(theta) * theta) / d) / t2
    return C * np.eye(3) + A * K + B * K2


def s_compose(a, b):
    """geometry.py:296-301"""
    qa, ta, sa = a
    qb, tb, sb = b
    return qcanon(qmul(qa, qb)), sa * (qmat(qa) @ tb) + ta, sa * sb


def s_inverse(a):
    """geometry.py:306-309 (Rotation.inverse canonicalises, geometry.py:169-171)"""
    q, t, s = a
    qi = qcanon(np.array([q[0], -q[1], -q[2], -q[3]]))
    inv_s = 1.0 / s
    return qi, -inv_s * (qmat(qi) @ t), inv_s


def s_exp(xi):
    """geometry.py:311-317"""
    omega, ups, sigma = xi[:3], xi[3:6], xi[6]
    return qexp(omega), sim3_w(omega, sigma) @ ups, float(np.exp(sigma))


def s_log(a):
    """geometry.py:319-324"""
    q, t, s = a
    omega = qlog(q)
    sigma = np.log(s)
    ups = np.linalg.solve(sim3_w(omega, sigma), t)
    return np.concatenate([omega, ups, [sigma]])


def s_adjoint(a):
    """geometry.py:329-339"""
    q, t, s = a
    R = qmat(q)
    A = np.zeros((7, 7))
    A[:3, :3] = R
    A[3:6, :3] = hat(t) @ R
    A[3:6, 3:6] = s * R
    A[3:6, 6] = -t
    A[6, 6] = 1.0
    return A


def sim3_ad(xi):
    """geometry.py:344-354"""
    omega, ups, sigma = xi[:3], xi[3:6], xi[6]
    A = np.zeros((7, 7))
    A[:3, :3] = hat(omega)
    A[3:6, :3] = hat(ups)
    A[3:6, 3:6] = hat(omega) + sigma * np.eye(3)
    A[3:6, 6] = -ups
    return A


def sim3_jr_inv(xi):
    """geometry.py:357-370: phi(-ad_xi) by the block-matrix exponential, inverted."""
    A = -sim3_ad(xi)
    M = np.zeros((14, 14))
    M[:7, :7] = A
    M[:7, 7:] = np.eye(7)
    return np.linalg.inv(expm(M)[:7, 7:])


def node_state(P, n):
    return np.asarray(P["sq"][n], float), np.asarray(P["st"][n], float), float(P["ss"][n])


def edge_state(P, r):
    return np.asarray(P["rq"][r], float), np.asarray(P["rt"][r], float), float(P["rs"][r])


# ----------------------------------------------------------------------------
# factors
# ----------------------------------------------------------------------------

def sim3_vision_residual(P, v, disp=None, states=None):
    """loopclosure.py:225-307 for vision loop edge ``v`` (rows scaled by sqrt(w))."""
    disp = P["disp"] if disp is None else disp
    S = P if states is None else states
    i, j = int(P["vi"][v]), int(P["vj"][v])
    r0, r1 = int(P["veoff"][v]), int(P["veoff"][v + 1])
    d = np.asarray(disp[P["doff"][i]:P["doff"][i + 1]], float)
    if len(d) != r1 - r0:
        raise ValueError("disparity length must match edge pixel list")
    if np.any(d <= 0.0):
        raise ValueError("disparities must be strictly positive")
    pix, tgt, wts = P["vpix"][r0:r1], P["vtgt"][r0:r1], P["vw"][r0:r1]
    fx, fy, cx, cy = P["intr"]
    R_bc, p_bc = _T_bc(P)
    qi, p_i, s_i = node_state(S, i)
    qj, p_j, s_j = node_state(S, j)
    R_i, R_j = qmat(qi), qmat(qj)
    n = len(d)
    z = 1.0 / d
    X_i = np.stack([(pix[:, 0] - cx) / fx * z, (pix[:, 1] - cy) / fy * z, z], axis=1)   # :245
    Y_i = X_i @ R_bc.T + p_bc
    X_w = s_i * (Y_i @ R_i.T) + p_i
    V_j = ((X_w - p_j) @ R_j) / s_j
    X_c = (V_j - p_bc) @ R_bc
    zz = X_c[:, 2]
    valid = zz > 1e-6
    zs = np.where(valid, zz, 1.0)
    pred = np.stack([fx * X_c[:, 0] / zs + cx, fy * X_c[:, 1] / zs + cy], axis=1)
    r = tgt - pred
    Pm = np.zeros((n, 2, 3))
    Pm[:, 0, 0] = fx / zs
    Pm[:, 0, 2] = -fx * X_c[:, 0] / zs ** 2
    Pm[:, 1, 1] = fy / zs
    Pm[:, 1, 2] = -fy * X_c[:, 1] / zs ** 2

    def hatr(vv):
        H = np.zeros((vv.shape[0], 3, 3))
        H[:, 0, 1], H[:, 0, 2] = -vv[:, 2], vv[:, 1]
        H[:, 1, 0], H[:, 1, 2] = vv[:, 2], -vv[:, 0]
        H[:, 2, 0], H[:, 2, 1] = -vv[:, 1], vv[:, 0]
        return H

    B = (R_bc.T @ R_j.T) / s_j                                       # :271-272
    BRi = B @ R_i
    dth_i = np.einsum("ab,nbc->nac", -s_i * BRi, hatr(Y_i))
    dp_i = np.broadcast_to(s_i * BRi, (n, 3, 3))
    ds_i = s_i * (Y_i @ BRi.T)
    dth_j = np.einsum("ab,nbc->nac", R_bc.T, hatr(V_j))
    dp_j = np.broadcast_to(-R_bc.T, (n, 3, 3))
    ds_j = -(V_j @ R_bc)
    C = s_i * (BRi @ R_bc)
    dd = -np.einsum("ab,nb->na", C, X_i) / d[:, None]
    J_i = np.concatenate([-np.einsum("nab,nbc->nac", Pm, dth_i), -np.einsum("nab,nbc->nac", Pm, dp_i),
                          -np.einsum("nab,nb->na", Pm, ds_i)[:, :, None]], axis=2)
    J_j = np.concatenate([-np.einsum("nab,nbc->nac", Pm, dth_j), -np.einsum("nab,nbc->nac", Pm, dp_j),
                          -np.einsum("nab,nb->na", Pm, ds_j)[:, :, None]], axis=2)
    J_d = -np.einsum("nab,nb->na", Pm, dd)
    sw = np.sqrt(np.where(valid[:, None], wts, 0.0))                   # :298-299
    return sw * r, sw[:, :, None] * J_i, sw[:, :, None] * J_j, sw * J_d, valid


def whitening(info):
    """residuals.py:370-377: W = L^T, L = cholesky(information) (symmetric-sqrt fallback)."""
    try:
        L = np.linalg.cholesky(info)
    except np.linalg.LinAlgError:
        vals, vecs = np.linalg.eigh(info)
        L = vecs @ np.diag(np.sqrt(np.maximum(vals, 0.0)))
    return L.T


def relative_pose_residual(P, r, states=None):
    """residuals.py:364-380 for relative edge ``r``: (whitened residual, J_i, J_j)."""
    S = P if states is None else states
    i, j = int(P["ri"][r]), int(P["rj"][r])
    Si, Sj = node_state(S, i), node_state(S, j)
    M = s_compose(s_compose(edge_state(P, r), Si), s_inverse(Sj))
    res = s_log(M)
    J_i = sim3_jr_inv(res) @ s_adjoint(Sj)
    W = whitening(np.asarray(P["rinfo"][r], float))
    return W @ res, W @ J_i, -(W @ J_i)


# ----------------------------------------------------------------------------
# solver (loopclosure.py:378-574)
# ----------------------------------------------------------------------------

def pg_energy(P):
    """loopclosure.py:378-390 (vision loops, then relative edges)."""
    e = 0.0
    for v in range(len(P["vi"])):
        e += float((sim3_vision_residual(P, v)[0] ** 2).sum())
    for r in range(len(P["ri"])):
        res = relative_pose_residual(P, r)[0]
        e += float(res @ res)
    return e


class PgLayout:
    """loopclosure.py:392-422: 7 dof per node, node 0 the gauge; disparity columns of
    vision-loop sources only (P['doff'] is that layout)."""

    def __init__(self, P, opts=None):
        self.K = len(P["kid"])
        self.sdof = SIM3_DOF
        self.npv = self.K * SIM3_DOF
        self.n_state = self.npv
        self.n_grav = 0
        self.doff = np.asarray(P["doff"], np.int64)
        self.n_disp = int(self.doff[-1])
        self.frozen = np.zeros(self.K, bool)
        self.frozen[0] = True

    def cols(self, n, a=0, b=SIM3_DOF):
        return np.arange(n * SIM3_DOF + a, n * SIM3_DOF + b)

    def free_mask(self):
        return np.repeat(~self.frozen, SIM3_DOF)


def linearize_pg(P, L):
    """loopclosure.py:425-475"""
    npv, nd = L.npv, L.n_disp
    H_pp = np.zeros((npv, npv))
    H_pd = np.zeros((npv, nd))
    H_dd = np.zeros(nd)
    g_p = np.zeros(npv)
    g_d = np.zeros(nd)

    def add_rel(i, j, r, Ji, Jj):
        ci, cj = L.cols(i), L.cols(j)
        H_pp[np.ix_(ci, ci)] += Ji.T @ Ji
        H_pp[np.ix_(cj, cj)] += Jj.T @ Jj
        Hij = Ji.T @ Jj
        H_pp[np.ix_(ci, cj)] += Hij
        H_pp[np.ix_(cj, ci)] += Hij.T
        g_p[ci] += Ji.T @ r
        g_p[cj] += Jj.T @ r

    for v in range(len(P["vi"])):
        i, j = int(P["vi"][v]), int(P["vj"][v])
        r, Ji, Jj, Jd, _ = sim3_vision_residual(P, v)
        ci, cj = L.cols(i), L.cols(j)
        cd = np.arange(L.doff[i], L.doff[i + 1])
        H_pp[np.ix_(ci, ci)] += np.einsum("nka,nkb->ab", Ji, Ji)
        H_pp[np.ix_(cj, cj)] += np.einsum("nka,nkb->ab", Jj, Jj)
        Hij = np.einsum("nka,nkb->ab", Ji, Jj)
        H_pp[np.ix_(ci, cj)] += Hij
        H_pp[np.ix_(cj, ci)] += Hij.T
        H_pd[np.ix_(ci, cd)] += np.einsum("nka,nk->na", Ji, Jd).T
        H_pd[np.ix_(cj, cd)] += np.einsum("nka,nk->na", Jj, Jd).T
        H_dd[cd] += np.einsum("nk,nk->n", Jd, Jd)
        g_p[ci] += np.einsum("nka,nk->a", Ji, r)
        g_p[cj] += np.einsum("nka,nk->a", Jj, r)
        g_d[cd] += np.einsum("nk,nk->n", Jd, r)
    for r in range(len(P["ri"])):
        res, Ji, Jj = relative_pose_residual(P, r)
        add_rel(int(P["ri"][r]), int(P["rj"][r]), res, Ji, Jj)
    return H_pp, H_pd, H_dd, g_p, g_d


def pg_apply(P, L, dx_full, dx_d):
    """loopclosure.py:489-499: free nodes S <- S exp(dx); disparities floored."""
    for n in range(L.K):
        if not L.frozen[n]:
            q, t, s = s_compose(node_state(P, n), s_exp(dx_full[n * SIM3_DOF:(n + 1) * SIM3_DOF]))
            P["sq"][n], P["st"][n], P["ss"][n] = q, t, s
        sl = slice(L.doff[n], L.doff[n + 1])
        if sl.stop > sl.start:
            P["disp"][sl] = np.maximum(P["disp"][sl] + dx_d[sl], DISPARITY_FLOOR)


_KEYS = ("sq", "st", "ss", "disp")


def solve_pgba(P, opts=None):
    """loopclosure.py:502-574 (LM over the pose graph; mutates P).  Returns the SolveReport
    fields; the LoopCorrection is formed by the caller from the before/after states."""
    from .vi_ba import DEFAULT_OPTS
    o = dict(DEFAULT_OPTS)
    o.update(opts or {})
    if int(P["n_loops"]) == 0:                                         # :510-513
        raise ValueError("pose graph has no loop edges")
    L = PgLayout(P)
    cost = pg_energy(P)
    if not np.isfinite(cost):
        raise RuntimeError("pose-graph energy is not finite")
    traj = [cost]
    lam = o["damping"]
    term = "max_iterations"
    iters = 0
    warns = []
    for it in range(o["max_iterations"]):
        lin = linearize_pg(P, L)
        accepted = False
        while True:
            try:
                dx, dxd = solve_step_dense(L, o, *lin, lam, o["use_schur"])
            except RuntimeError as exc:
                warns.append(str(exc))
                lam *= o["damping_up"]
                if lam > o["max_damping"]:
                    return dict(iterations=iters, initial_cost=traj[0], final_cost=cost, cost_trajectory=traj,
                                termination=f"singular: {exc}", condition_warnings=warns)
                continue
            snap = {k: np.array(P[k], copy=True) for k in _KEYS}
            pg_apply(P, L, dx, dxd)
            new = pg_energy(P)
            if np.isfinite(new) and new < cost:
                cost = new
                traj.append(cost)
                lam = max(lam * o["damping_down"], 1e-12)
                accepted = True
                iters = it + 1
                step_inf = max(np.max(np.abs(dx), initial=0.0), np.max(np.abs(dxd), initial=0.0))
                if step_inf < o["step_tol"]:
                    term = "converged"
                break
            for k, v in snap.items():
                P[k] = v
            lam *= o["damping_up"]
            if lam > o["max_damping"]:
                term = "no_decrease_at_max_damping"
                break
        if not accepted:
            break
        if term == "converged":
            break
        prev = traj[-2]
        if prev > 0 and (prev - cost) / prev < o["rel_decrease_tol"]:
            term = "converged"
            break
    else:
        term = "max_iterations"
    return dict(iterations=iters, initial_cost=traj[0], final_cost=cost, cost_trajectory=traj,
                termination=term, condition_warnings=warns)


def clone(P):
    return copy.deepcopy(P)
