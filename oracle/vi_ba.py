"""fp64 numpy restatement of the reference VI-BA path — TEST INFRASTRUCTURE.

Every function cites the reference lines it restates (paths relative to
/root/reference/pkg/src/vislam/).  Inputs are the *packed problem* dict used
across this repo (documented in DESIGN.md §3 and produced by
``paper_2512_02293_b200.problem.pack_graph``):

  q[K,4] p[K,3] v[K,3] bg[K,3] ba[K,3] ts[K] kid[K]      keyframe states (fp64)
  doff[K+1] disp[n_disp]                                  per-keyframe disparities
  ei[E] ej[E] eoff[E+1] epix[R,2] tgt[R,2] w[R,2]         vision edges (keyframe *indices*)
  fi[F] fj[F] f_dt f_dR[F,4] f_dp f_dv f_Jr[F,3,3]        preintegrated IMU factors
  f_Jp[F,3,6] f_Jv[F,3,6] f_cov[F,15,15] f_bhat[F,6]
  grav_q[4] grav_G  intr[4]=(fx,fy,cx,cy)  Tcb[7]=(q,t)  has_Tcb

The oracle never runs inside the product; see oracle/__init__.py.
"""

from __future__ import annotations

import copy

import numpy as np

SMALL_ANGLE = 1e-8          # geometry.py:20
DISPARITY_FLOOR = 1e-4      # solver.py:32
STATE_DOF = 15              # solver.py:33
POSE_DOF = 6                # solver.py:34
GRAV_BASIS = np.array([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]])   # residuals.py:141


# ----------------------------------------------------------------------------
# SO(3) / quaternion maps  (geometry.py:23-184)
# ----------------------------------------------------------------------------

def hat(v):
    """geometry.py:23-30"""
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def so3_exp_matrix(w):
    """geometry.py:33-43 (second-order Taylor below the cutoff)."""
    th = np.linalg.norm(w)
    K = hat(w)
    if th < SMALL_ANGLE:
        return np.eye(3) + K + 0.5 * (K @ K)
    return np.eye(3) + (np.sin(th) / th) * K + ((1.0 - np.cos(th)) / (th * th)) * (K @ K)


def so3_jr(w):
    """geometry.py:57-67"""
    th = np.linalg.norm(w)
    K = hat(w)
    if th < SMALL_ANGLE:
        return np.eye(3) - 0.5 * K + (K @ K) / 6.0
    t2 = th * th
    return np.eye(3) - ((1.0 - np.cos(th)) / t2) * K + ((th - np.sin(th)) / (t2 * th)) * (K @ K)


def so3_jr_inv(w):
    """geometry.py:70-80"""
    th = np.linalg.norm(w)
    K = hat(w)
    if th < SMALL_ANGLE:
        return np.eye(3) + 0.5 * K + (K @ K) / 12.0
    b = (1.0 / (th * th)) * (1.0 - th * (1.0 / np.tan(0.5 * th)) / 2.0)
    return np.eye(3) + 0.5 * K + b * (K @ K)


def qmul(a, b):
    """geometry.py:83-91 (Hamilton product, wxyz)."""
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def qcanon(q):
    """geometry.py:94-98 — unit norm, w >= 0."""
    q = q / np.linalg.norm(q)
    return -q if q[0] < 0.0 else q


def qmat(q):
    """geometry.py:151-157"""
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def qexp(w):
    """geometry.py:113-123 (first-order quaternion below the cutoff)."""
    th = np.linalg.norm(w)
    if th < SMALL_ANGLE:
        return qcanon(np.concatenate(([1.0], 0.5 * w)))
    return qcanon(np.concatenate(([np.cos(0.5 * th)], np.sin(0.5 * th) * (w / th))))


def qfrom_matrix(R):
    """geometry.py:125-149 (trace / largest-diagonal branches)."""
    t = np.trace(R)
    if t > 0.0:
        s = np.sqrt(t + 1.0) * 2.0
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
    else:
        i = int(np.argmax(np.diag(R)))
        if i == 0:
            s = np.sqrt(1.0 + R[0, 0] - R[1, 1] - R[2, 2]) * 2.0
            q = [(R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s]
        elif i == 1:
            s = np.sqrt(1.0 + R[1, 1] - R[0, 0] - R[2, 2]) * 2.0
            q = [(R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s]
        else:
            s = np.sqrt(1.0 + R[2, 2] - R[0, 0] - R[1, 1]) * 2.0
            q = [(R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s]
    return qcanon(np.array(q))


def qlog(q):
    """geometry.py:159-167"""
    w, v = q[0], q[1:]
    n = np.linalg.norm(v)
    if n < SMALL_ANGLE:
        return (2.0 / w) * v
    return (2.0 * np.arctan2(n, w) / n) * v


# ----------------------------------------------------------------------------
# factors  (residuals.py:172-354)
# ----------------------------------------------------------------------------

def _T_bc(P):
    """residuals.py:187-192 — T_bc = T_cb^{-1} (identity when T_cb is None)."""
    if not bool(P.get("has_Tcb", False)):
        return np.eye(3), np.zeros(3)
    q = np.asarray(P["Tcb"][:4], float)
    t = np.asarray(P["Tcb"][4:7], float)
    qi = qcanon(np.array([q[0], -q[1], -q[2], -q[3]]))      # geometry.py:169-171
    Ri = qmat(qi)
    return Ri, -(Ri @ t)                                       # geometry.py:217-219


def vision_residual(P, e, disp=None):
    """residuals.py:172-263 for edge ``e`` of the packed problem.

    Returns (r, J_i, J_j, J_d, valid) with rows scaled by sqrt(w), w zeroed on
    invalid (behind-camera) pixels.  Huber is never used by the solver.
    """
    disp = P["disp"] if disp is None else disp
    i, j = int(P["ei"][e]), int(P["ej"][e])
    r0, r1 = int(P["eoff"][e]), int(P["eoff"][e + 1])
    d = disp[P["doff"][i]:P["doff"][i + 1]]
    if len(d) != r1 - r0:
        raise ValueError("disparity length must match edge pixel list")
    if np.any(d <= 0.0):
        raise ValueError("disparities must be strictly positive")
    pix, tgt, wts = P["epix"][r0:r1], P["tgt"][r0:r1], P["w"][r0:r1]
    fx, fy, cx, cy = P["intr"]
    R_bc, p_bc = _T_bc(P)
    R_i, p_i = qmat(P["q"][i]), P["p"][i]
    R_j, p_j = qmat(P["q"][j]), P["p"][j]
    n = len(d)

    z = 1.0 / d                                                   # backproject :81-87
    X_i = np.stack([(pix[:, 0] - cx) / fx * z, (pix[:, 1] - cy) / fy * z, z], axis=1)
    Y_i = X_i @ R_bc.T + p_bc                                      # :200
    X_w = Y_i @ R_i.T + p_i                                        # :201
    R_cw_j = R_bc.T @ R_j.T                                        # :202
    V_j = X_w - p_j                                                # :203
    X_j = V_j @ (R_j @ R_bc) - R_bc.T @ p_bc                       # :204

    zz = X_j[:, 2]
    valid = zz > 1e-6                                              # :206-209
    zs = np.where(valid, zz, 1.0)
    pred = np.stack([fx * X_j[:, 0] / zs + cx, fy * X_j[:, 1] / zs + cy], axis=1)
    r = tgt - pred                                                 # :213

    Pm = np.zeros((n, 2, 3))                                       # :216-220
    Pm[:, 0, 0] = fx / zs
    Pm[:, 0, 2] = -fx * X_j[:, 0] / zs ** 2
    Pm[:, 1, 1] = fy / zs
    Pm[:, 1, 2] = -fy * X_j[:, 1] / zs ** 2

    def hatb(vv):
        H = np.zeros((vv.shape[0], 3, 3))
        H[:, 0, 1], H[:, 0, 2] = -vv[:, 2], vv[:, 1]
        H[:, 1, 0], H[:, 1, 2] = vv[:, 2], -vv[:, 0]
        H[:, 2, 0], H[:, 2, 1] = -vv[:, 1], vv[:, 0]
        return H

    dth_i = np.einsum("ab,nbc->nac", -R_cw_j @ R_i, hatb(Y_i))     # :233
    dth_j = np.einsum("ab,nbc->nac", R_bc.T, hatb(V_j @ R_j))      # :235
    dd = -np.einsum("ab,nb->na", R_cw_j @ R_i @ R_bc, X_i) / d[:, None]   # :237
    J_i = np.concatenate([-np.einsum("nab,nbc->nac", Pm, dth_i),
                          -np.einsum("nab,bc->nac", Pm, R_cw_j)], axis=2)   # :239-242
    J_j = np.concatenate([-np.einsum("nab,nbc->nac", Pm, dth_j),
                          np.einsum("nab,bc->nac", Pm, R_cw_j)], axis=2)    # :243-246
    J_d = -np.einsum("nab,nb->na", Pm, dd)                          # :247

    sw = np.sqrt(np.where(valid[:, None], wts, 0.0))                # :249-254
    return sw * r, sw[:, :, None] * J_i, sw[:, :, None] * J_j, sw * J_d, valid


def _chol_lower(A):
    """scipy.linalg.cholesky(lower=True) as used at residuals.py:338-341."""
    try:
        return np.linalg.cholesky(A)
    except np.linalg.LinAlgError as exc:
        raise ValueError("non-PSD preintegration covariance") from exc


def _fwd_subst(L, B):
    """solve_triangular(L, B, lower=True) (residuals.py:345-346)."""
    n = L.shape[0]
    X = np.array(B, dtype=float, copy=True)
    for r in range(n):
        X[r] = (X[r] - L[r, :r] @ X[:r]) / L[r, r]
    return X


def inertial_residual(P, f, state=None):
    """residuals.py:274-354 for IMU factor ``f``; returns (r, J_i, J_j, J_g)."""
    S = P if state is None else state
    i, j = int(P["fi"][f]), int(P["fj"][f])
    dt = S["ts"][j] - S["ts"][i] if "ts" in S else P["ts"][j] - P["ts"][i]
    if abs(dt - P["f_dt"][f]) > 1e-6:                              # :281-284
        raise ValueError("delta spans %.6fs but states are %.6fs apart" % (P["f_dt"][f], dt))
    R_i, R_j = qmat(S["q"][i]), qmat(S["q"][j])
    p_i, p_j, v_i, v_j = S["p"][i], S["p"][j], S["v"][i], S["v"][j]
    b_i = np.concatenate([S["bg"][i], S["ba"][i]])
    b_j = np.concatenate([S["bg"][j], S["ba"][j]])
    R_wg = qmat(S["grav_q"])
    gI = np.array([0.0, 0.0, float(S["grav_G"])])
    g = gI @ R_wg.T                                                # residuals.py:125-130
    db = b_i - P["f_bhat"][f]
    dbg = db[:3]
    Jr_, Jp_, Jv_ = P["f_Jr"][f], P["f_Jp"][f], P["f_Jv"][f]

    ct = Jr_ @ dbg                                                  # :294-296
    C = qmat(P["f_dR"][f]) @ so3_exp_matrix(ct)
    r_rot = qlog(qfrom_matrix(C.T @ R_i.T @ R_j))
    s_pos = p_j - p_i - v_i * dt - 0.5 * dt * dt * g                # :297-300
    r_pos = R_i.T @ s_pos - (P["f_dp"][f] + Jp_ @ db)
    s_vel = v_j - v_i - dt * g
    r_vel = R_i.T @ s_vel - (P["f_dv"][f] + Jv_ @ db)
    r_bias = b_j - b_i

    Jri = so3_jr_inv(r_rot)                                         # :303-304
    Jli = so3_jr_inv(-r_rot)
    J_i = np.zeros((15, 15))
    J_j = np.zeros((15, 15))
    J_g = np.zeros((15, 3))
    J_i[0:3, 0:3] = -Jri @ (R_j.T @ R_i)                            # :310-313
    J_j[0:3, 0:3] = Jri
    J_i[0:3, 9:12] = -Jli @ so3_jr(ct) @ Jr_
    J_i[3:6, 0:3] = hat(R_i.T @ s_pos)                              # :315-321
    J_i[3:6, 3:6] = -R_i.T
    J_j[3:6, 3:6] = R_i.T
    J_i[3:6, 6:9] = -dt * R_i.T
    J_i[3:6, 9:15] = -Jp_
    J_g[3:6, :] = 0.5 * dt * dt * R_i.T @ R_wg @ hat(gI)
    J_i[6:9, 0:3] = hat(R_i.T @ s_vel)                              # :323-328
    J_i[6:9, 6:9] = -R_i.T
    J_j[6:9, 6:9] = R_i.T
    J_i[6:9, 9:15] = -Jv_
    J_g[6:9, :] = dt * R_i.T @ R_wg @ hat(gI)
    J_i[9:15, 9:15] = -np.eye(6)                                    # :330-332
    J_j[9:15, 9:15] = np.eye(6)

    r = np.concatenate([r_rot, r_pos, r_vel, r_bias])
    cov = P["f_cov"][f]
    L9 = _chol_lower(cov[:9, :9])                                   # :335-341
    Lb = _chol_lower(cov[9:15, 9:15])

    def whiten(M):                                                  # :343-347
        M = M.reshape(15, -1)
        out = np.empty_like(M)
        out[:9] = _fwd_subst(L9, M[:9])
        out[9:] = _fwd_subst(Lb, M[9:])
        return out

    return whiten(r).reshape(15), whiten(J_i), whiten(J_j), whiten(J_g)


# ----------------------------------------------------------------------------
# solver  (solver.py:118-411)
# ----------------------------------------------------------------------------

def total_energy(P, parts=False):
    """solver.py:118-131 — Σ whitened squared residuals."""
    ev = 0.0
    for e in range(len(P["ei"])):
        r = vision_residual(P, e)[0]
        ev += float((r ** 2).sum())
    ei = 0.0
    for f in range(len(P["fi"])):
        r = inertial_residual(P, f)[0]
        ei += float((r ** 2).sum())
    return (ev, ei) if parts else ev + ei


class Layout:
    """solver.py:139-170 — column bookkeeping (frozen by kid)."""

    def __init__(self, P, opts):
        self.K = len(P["kid"])
        frozen = set(int(k) for k in opts.get("frozen_keyframes", (0,)))
        self.frozen = np.array([int(k) in frozen for k in P["kid"]])
        self.sdof = STATE_DOF if opts.get("optimize_velocity_bias", True) else POSE_DOF
        self.n_state = self.K * self.sdof
        self.n_grav = 2 if opts.get("optimize_gravity", False) else 0
        self.npv = self.n_state + self.n_grav
        self.doff = np.asarray(P["doff"], dtype=np.int64)
        self.n_disp = int(self.doff[-1])

    def cols(self, n, a, b):
        return np.arange(n * self.sdof + a, n * self.sdof + b)

    def free_mask(self):
        m = np.ones(self.npv, dtype=bool)
        for n in range(self.K):
            if self.frozen[n]:
                m[n * self.sdof:(n + 1) * self.sdof] = False
        return m


def _imu_blocks(P, L, f):
    r, Ji, Jj, Jg = inertial_residual(P, f)
    return r, Ji[:, :L.sdof], Jj[:, :L.sdof], Jg @ GRAV_BASIS


def linearize_dense(P, L):
    """solver.py:173-251 verbatim in structure (dense H_pd: small problems)."""
    npv, nd, sd = L.npv, L.n_disp, L.sdof
    H_pp = np.zeros((npv, npv))
    H_pd = np.zeros((npv, nd))
    H_dd = np.zeros(nd)
    g_p = np.zeros(npv)
    g_d = np.zeros(nd)
    for e in range(len(P["ei"])):
        i, j = int(P["ei"][e]), int(P["ej"][e])
        r, Ji, Jj, Jd, _ = vision_residual(P, e)
        ci, cj = L.cols(i, 0, 6), L.cols(j, 0, 6)
        cd = np.arange(L.doff[i], L.doff[i + 1])
        Hij = np.einsum("nka,nkb->ab", Ji, Jj)
        H_pp[np.ix_(ci, ci)] += np.einsum("nka,nkb->ab", Ji, Ji)
        H_pp[np.ix_(cj, cj)] += np.einsum("nka,nkb->ab", Jj, Jj)
        H_pp[np.ix_(ci, cj)] += Hij
        H_pp[np.ix_(cj, ci)] += Hij.T
        H_pd[np.ix_(ci, cd)] += np.einsum("nka,nk->na", Ji, Jd).T
        H_pd[np.ix_(cj, cd)] += np.einsum("nka,nk->na", Jj, Jd).T
        H_dd[cd] += np.einsum("nk,nk->n", Jd, Jd)
        g_p[ci] += np.einsum("nka,nk->a", Ji, r)
        g_p[cj] += np.einsum("nka,nk->a", Jj, r)
        g_d[cd] += np.einsum("nk,nk->n", Jd, r)
    gc = np.arange(L.n_state, L.n_state + L.n_grav)
    for f in range(len(P["fi"])):
        i, j = int(P["fi"][f]), int(P["fj"][f])
        r, Ji, Jj, Jg = _imu_blocks(P, L, f)
        ci, cj = L.cols(i, 0, sd), L.cols(j, 0, sd)
        H_pp[np.ix_(ci, ci)] += Ji.T @ Ji
        H_pp[np.ix_(cj, cj)] += Jj.T @ Jj
        H_pp[np.ix_(ci, cj)] += Ji.T @ Jj
        H_pp[np.ix_(cj, ci)] += (Ji.T @ Jj).T
        g_p[ci] += Ji.T @ r
        g_p[cj] += Jj.T @ r
        if L.n_grav:
            H_pp[np.ix_(gc, gc)] += Jg.T @ Jg
            H_pp[np.ix_(ci, gc)] += Ji.T @ Jg
            H_pp[np.ix_(gc, ci)] += (Ji.T @ Jg).T
            H_pp[np.ix_(cj, gc)] += Jj.T @ Jg
            H_pp[np.ix_(gc, cj)] += (Jj.T @ Jg).T
            g_p[gc] += Jg.T @ r
    return H_pp, H_pd, H_dd, g_p, g_d


def linearize_sparse(P, L):
    """Same sums as linearize_dense, H_pd kept per source keyframe.

    Returns (H_pp, Hpd_blocks, H_dd, g_p, g_d) where Hpd_blocks[n] is a dict
    {keyframe index -> (6, N_n) coupling of that pose with keyframe n's
    disparities} (solver.py:209-214 without the dense scatter).
    """
    npv, nd, sd = L.npv, L.n_disp, L.sdof
    H_pp = np.zeros((npv, npv))
    H_dd = np.zeros(nd)
    g_p = np.zeros(npv)
    g_d = np.zeros(nd)
    Hpd = [dict() for _ in range(L.K)]
    for e in range(len(P["ei"])):
        i, j = int(P["ei"][e]), int(P["ej"][e])
        r, Ji, Jj, Jd, _ = vision_residual(P, e)
        ci, cj = L.cols(i, 0, 6), L.cols(j, 0, 6)
        sl = slice(L.doff[i], L.doff[i + 1])
        Hij = np.einsum("nka,nkb->ab", Ji, Jj)
        H_pp[np.ix_(ci, ci)] += np.einsum("nka,nkb->ab", Ji, Ji)
        H_pp[np.ix_(cj, cj)] += np.einsum("nka,nkb->ab", Jj, Jj)
        H_pp[np.ix_(ci, cj)] += Hij
        H_pp[np.ix_(cj, ci)] += Hij.T
        for kf, J in ((i, Ji), (j, Jj)):
            blk = np.einsum("nka,nk->an", J, Jd)
            Hpd[i][kf] = Hpd[i][kf] + blk if kf in Hpd[i] else blk
        H_dd[sl] += np.einsum("nk,nk->n", Jd, Jd)
        g_p[ci] += np.einsum("nka,nk->a", Ji, r)
        g_p[cj] += np.einsum("nka,nk->a", Jj, r)
        g_d[sl] += np.einsum("nk,nk->n", Jd, r)
    H_imu, g_imu = _imu_part(P, L)
    return H_pp + H_imu, Hpd, H_dd, g_p + g_imu, g_d


def _imu_part(P, L):
    npv, sd = L.npv, L.sdof
    H = np.zeros((npv, npv))
    g = np.zeros(npv)
    gc = np.arange(L.n_state, L.n_state + L.n_grav)
    for f in range(len(P["fi"])):
        i, j = int(P["fi"][f]), int(P["fj"][f])
        r, Ji, Jj, Jg = _imu_blocks(P, L, f)
        ci, cj = L.cols(i, 0, sd), L.cols(j, 0, sd)
        H[np.ix_(ci, ci)] += Ji.T @ Ji
        H[np.ix_(cj, cj)] += Jj.T @ Jj
        H[np.ix_(ci, cj)] += Ji.T @ Jj
        H[np.ix_(cj, ci)] += (Ji.T @ Jj).T
        g[ci] += Ji.T @ r
        g[cj] += Jj.T @ r
        if L.n_grav:
            H[np.ix_(gc, gc)] += Jg.T @ Jg
            H[np.ix_(ci, gc)] += Ji.T @ Jg
            H[np.ix_(gc, ci)] += (Ji.T @ Jg).T
            H[np.ix_(cj, gc)] += Jj.T @ Jg
            H[np.ix_(gc, cj)] += (Jj.T @ Jg).T
            g[gc] += Jg.T @ r
    return H, g


def _damp(diag, lam, ridge):
    """solver.py:260-262"""
    return diag * (1.0 + lam) + ridge


def solve_step_dense(L, opts, H_pp, H_pd, H_dd, g_p, g_d, lam, use_schur=True):
    """solver.py:254-308 (Schur path and the dense reference path)."""
    free = L.free_mask()
    Hf = H_pp[np.ix_(free, free)].copy()
    Hfd = H_pd[free]
    gf = g_p[free]
    nf, nd = Hf.shape[0], L.n_disp
    ridge = opts.get("ridge", 1e-10)
    idx = np.arange(nf)
    Hf[idx, idx] = _damp(np.diag(Hf), lam, ridge)
    Hdd = _damp(H_dd, lam, ridge)
    if use_schur and nd:
        inv = 1.0 / Hdd
        Hred = Hf - (Hfd * inv) @ Hfd.T
        gred = gf - Hfd @ (inv * g_d)
        try:
            dxf = np.linalg.solve(Hred, -gred)
        except np.linalg.LinAlgError as exc:
            raise RuntimeError("singular reduced pose system") from exc
        dxd = inv * (-g_d - Hfd.T @ dxf)
    else:
        n = nf + nd
        H = np.zeros((n, n))
        H[:nf, :nf] = Hf
        if nd:
            H[:nf, nf:] = Hfd
            H[nf:, :nf] = Hfd.T
            H[nf + np.arange(nd), nf + np.arange(nd)] = Hdd
        try:
            dx = np.linalg.solve(H, -np.concatenate([gf, g_d]))
        except np.linalg.LinAlgError as exc:
            raise RuntimeError("singular full system") from exc
        dxf, dxd = dx[:nf], dx[nf:]
    dx_full = np.zeros(L.npv)
    dx_full[free] = dxf
    return dx_full, dxd


def reduced_system_sparse(L, opts, H_pp, Hpd, H_dd, g_p, g_d, lam):
    """Schur complement of solver.py:276-285 accumulated per source keyframe.

    Algebraically identical to ``Hf_d - (Hfd*inv_dd) @ Hfd.T``: every
    disparity column couples only the poses of its own keyframe's edges, so
    the fill-in is a sum of per-keyframe dense products.  Returns the full
    (npv) damped-and-reduced system before freezing, and inv_dd.
    """
    ridge = opts.get("ridge", 1e-10)
    H = H_pp.copy()
    idx = np.arange(L.npv)
    H[idx, idx] = _damp(np.diag(H_pp), lam, ridge)
    g = g_p.copy()
    inv = 1.0 / _damp(H_dd, lam, ridge)
    for n in range(L.K):
        if not Hpd[n]:
            continue
        sl = slice(L.doff[n], L.doff[n + 1])
        kfs = sorted(Hpd[n])
        cols = np.concatenate([L.cols(k, 0, 6) for k in kfs])
        B = np.concatenate([Hpd[n][k] for k in kfs], axis=0)     # (6m, N_n)
        H[np.ix_(cols, cols)] -= (B * inv[sl]) @ B.T
        g[cols] -= B @ (inv[sl] * g_d[sl])
    return H, g, inv


def solve_step_sparse(L, opts, H_pp, Hpd, H_dd, g_p, g_d, lam):
    """solver.py:265-308 (Schur path) using the per-keyframe fill-in."""
    H, g, inv = reduced_system_sparse(L, opts, H_pp, Hpd, H_dd, g_p, g_d, lam)
    free = L.free_mask()
    try:
        dxf = np.linalg.solve(H[np.ix_(free, free)], -g[free])
    except np.linalg.LinAlgError as exc:
        raise RuntimeError("singular reduced pose system") from exc
    dx_full = np.zeros(L.npv)
    dx_full[free] = dxf
    dxd = inv * (-g_d)
    for n in range(L.K):
        if not Hpd[n]:
            continue
        sl = slice(L.doff[n], L.doff[n + 1])
        acc = -g_d[sl].copy()
        for k in sorted(Hpd[n]):
            acc -= Hpd[n][k].T @ dx_full[L.cols(k, 0, 6)]
        dxd[sl] = inv[sl] * acc
    return dx_full, dxd


def apply_step(P, L, dx_full, dx_d):
    """solver.py:326-341 with PoseState.retract (residuals.py:44-52) and
    Pose.retract (geometry.py:221-223).  Mutates P."""
    sd = L.sdof
    for n in range(L.K):
        seg = dx_full[n * sd:(n + 1) * sd]
        P["q"][n] = qcanon(qmul(P["q"][n], qexp(seg[0:3])))
        P["p"][n] = P["p"][n] + seg[3:6]
        if sd == STATE_DOF:
            P["v"][n] = P["v"][n] + seg[6:9]
            P["bg"][n] = P["bg"][n] + seg[9:12]
            P["ba"][n] = P["ba"][n] + seg[12:15]
        sl = slice(L.doff[n], L.doff[n + 1])
        if sl.stop > sl.start:
            P["disp"][sl] = np.maximum(P["disp"][sl] + dx_d[sl], DISPARITY_FLOOR)
    if L.n_grav:
        dg = GRAV_BASIS @ dx_full[L.n_state:L.n_state + 2]
        P["grav_q"] = qcanon(qmul(P["grav_q"], qexp(dg)))          # residuals.py:132-134


_STATE_KEYS = ("q", "p", "v", "bg", "ba", "disp", "grav_q")


def _snapshot(P):
    """solver.py:311-315"""
    return {k: np.array(P[k], copy=True) for k in _STATE_KEYS}


def _restore(P, snap):
    """solver.py:318-323"""
    for k, v in snap.items():
        P[k] = v


DEFAULT_OPTS = dict(max_iterations=10, damping=1e-4, damping_up=10.0, damping_down=0.5,
                    rel_decrease_tol=1e-8, step_tol=1e-10, max_damping=1e8,
                    frozen_keyframes=(0,), optimize_gravity=False,
                    optimize_velocity_bias=True, use_schur=True, ridge=1e-10)


def solve_vi_ba(P, opts=None, sparse=None):
    """solver.py:344-411 — LM driver.  Mutates P in place, returns a report
    dict with the SolveReport fields (solver.py:108-115)."""
    o = dict(DEFAULT_OPTS)
    o.update(opts or {})
    L = Layout(P, o)
    if sparse is None:
        sparse = L.npv * max(L.n_disp, 1) > 4e7
    cost = total_energy(P)
    traj = [cost]
    if o["max_iterations"] == 0:
        return dict(iterations=0, initial_cost=cost, final_cost=cost, cost_trajectory=traj,
                    termination="max_iterations", condition_warnings=[])
    lam = o["damping"]
    term = "max_iterations"
    iters = 0
    warns = []
    for it in range(o["max_iterations"]):
        if sparse:
            lin = linearize_sparse(P, L)
        else:
            lin = linearize_dense(P, L)
        accepted = False
        while True:
            try:
                if sparse:
                    dx, dxd = solve_step_sparse(L, o, *lin, lam)
                else:
                    dx, dxd = solve_step_dense(L, o, *lin, lam, o["use_schur"])
            except RuntimeError as exc:
                warns.append(str(exc))
                lam *= o["damping_up"]
                if lam > o["max_damping"]:
                    return dict(iterations=iters, initial_cost=traj[0], final_cost=cost,
                                cost_trajectory=traj, termination=f"singular: {exc}",
                                condition_warnings=warns)
                continue
            snap = _snapshot(P)
            apply_step(P, L, dx, dxd)
            new = total_energy(P)
            if new < cost:
                cost = new
                traj.append(cost)
                lam = max(lam * o["damping_down"], 1e-12)
                accepted = True
                iters = it + 1
                step_inf = max(np.max(np.abs(dx), initial=0.0), np.max(np.abs(dxd), initial=0.0))
                if step_inf < o["step_tol"]:
                    term = "converged"
                break
            _restore(P, snap)
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
