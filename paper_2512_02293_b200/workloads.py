"""Seeded synthetic VI-BA windows with the shapes of BASELINE.json configs 0-4.

The paper's datasets are not available here; these inputs stand in for them
with BASELINE.json's shapes and distributions (SURVEY.md §8(d) pins the
choices BASELINE leaves open):

* keyframes at 10 Hz, IMU at 200 Hz (20 intervals per keyframe pair);
* a looping trajectory (1 m/s on a ~1.15 m circle, 72 keyframes = 5° yaw per step)
  with a smooth 3° orientation wobble, so keyframes more than 30 apart
  revisit the same place and loop edges are covisible;
* IMU white noise σ_gyro=0.002, σ_acc=0.02 per sample and a bias random walk
  (densities 1e-5 / 1e-4); keyframe states come from midpoint integration of
  the clean signal, so the inertial residual at truth is the noise only;
* per-keyframe dense H×W pixel grid, depth ~ U[0.5, 5] m, disparity = 1/depth;
* directed edges: nearest-by-index proximity graph plus covisible loop edges
  (|i-j| > 30, true relative pose within 0.3 m / 15°);
* targets = true reprojection + N(0, σ) (cfg 2: σ=1 px, 10 % outliers offset
  U(±20) px with weight 0.05), weights U(0, 1); pixels whose true point has
  z <= 0.05 m in the target camera get weight 0 (synth.py:553-569 convention);
* initial estimate: truth perturbed by 2° / 0.05 m / 0.02 m/s (keyframe 0
  frozen, windows.py:164-177), disparities × U(0.97, 1.03), bias states =
  preintegration linearisation point b̂ = truth + N(0, 1e-3).

All per-pixel inputs are rounded to fp32 so the GPU path (fp32 storage) and
the CPU reference see identical values.  ``make_workload`` returns a
``FrameGraph`` of ``paper_2512_02293_b200.types`` objects plus the iteration
count BASELINE.json assigns to the config.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import types as T


@dataclass(frozen=True)
class ConfigSpec:
    n_kf: int
    grid: tuple          # (rows, cols)
    n_edges: int
    n_loop: int
    iterations: int
    sigma_px: float = 0.5
    outlier_rate: float = 0.0
    intr_scale: float = 1.0


CONFIGS = {
    0: ConfigSpec(8, (48, 64), 24, 0, 2),
    1: ConfigSpec(16, (48, 64), 96, 0, 4),
    2: ConfigSpec(16, (96, 128), 160, 0, 4, sigma_px=1.0, outlier_rate=0.10, intr_scale=2.0),
    3: ConfigSpec(128, (48, 64), 2048, 200, 3),
    4: ConfigSpec(512, (48, 64), 12288, 1000, 2),
}

KF_DT = 0.1
IMU_STEPS = 20
GRAVITY = 9.81
LAP_KF = 72            # 5° of yaw per keyframe step
FX_FULL = 320.0
SIGMA_GYRO = 0.002
SIGMA_ACC = 0.02
RATE = IMU_STEPS / KF_DT


# --------------------------------------------------------------------------
# small SO(3) helpers (batched)
# --------------------------------------------------------------------------

def _hat(v):
    v = np.asarray(v)
    H = np.zeros(v.shape[:-1] + (3, 3))
    H[..., 0, 1], H[..., 0, 2] = -v[..., 2], v[..., 1]
    H[..., 1, 0], H[..., 1, 2] = v[..., 2], -v[..., 0]
    H[..., 2, 0], H[..., 2, 1] = -v[..., 1], v[..., 0]
    return H


def _exp(w):
    """Rodrigues (batched)."""
    th = np.linalg.norm(w, axis=-1)[..., None, None]
    K = _hat(w)
    K2 = K @ K
    small = th < 1e-8
    ths = np.where(small, 1.0, th)
    a = np.where(small, 1.0, np.sin(ths) / ths)
    b = np.where(small, 0.5, (1.0 - np.cos(ths)) / (ths * ths))
    return np.eye(3) + a * K + b * K2


def _jr(w):
    th = np.linalg.norm(w, axis=-1)[..., None, None]
    K = _hat(w)
    K2 = K @ K
    small = th < 1e-8
    ths = np.where(small, 1.0, th)
    a = np.where(small, 0.5, (1.0 - np.cos(ths)) / (ths * ths))
    b = np.where(small, 1.0 / 6.0, (ths - np.sin(ths)) / (ths ** 3))
    return np.eye(3) - a * K + b * K2


def _rz(phi):
    c, s = np.cos(phi), np.sin(phi)
    R = np.zeros(np.shape(phi) + (3, 3))
    R[..., 0, 0], R[..., 0, 1] = c, -s
    R[..., 1, 0], R[..., 1, 1] = s, c
    R[..., 2, 2] = 1.0
    return R


_R0 = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])   # camera looks radially out


class _Motion:
    """Analytic looping motion: R(t) = Rz(Ωt) R0 Exp(θ(t)), p(t) = circle + wobble."""

    def __init__(self, rng):
        self.Om = 2.0 * np.pi / (LAP_KF * KF_DT)
        self.rho = 1.0 / self.Om
        # wobble frequencies are integer multiples of the lap frequency, so a
        # revisit one lap later reproduces the pose (covisible loop edges)
        flap = 1.0 / (LAP_KF * KF_DT)
        self.A = np.deg2rad(3.0) * rng.uniform(0.5, 1.0, 3)
        self.f = flap * rng.integers(1, 4, 3)
        self.ph = rng.uniform(0, 2 * np.pi, 3)
        self.B = 0.02 * rng.uniform(0.5, 1.0, 3)
        self.g = flap * rng.integers(1, 4, 3)
        self.ps = rng.uniform(0, 2 * np.pi, 3)

    def theta(self, t):
        return self.A * np.sin(2 * np.pi * self.f * t[:, None] + self.ph)

    def theta_dot(self, t):
        return self.A * 2 * np.pi * self.f * np.cos(2 * np.pi * self.f * t[:, None] + self.ph)

    def R(self, t):
        return _rz(self.Om * t) @ _R0 @ _exp(self.theta(t))

    def p(self, t):
        ph = self.Om * t
        return (np.stack([self.rho * np.cos(ph), self.rho * np.sin(ph), 0 * t], 1)
                + self.B * np.sin(2 * np.pi * self.g * t[:, None] + self.ps))

    def v(self, t):
        ph = self.Om * t
        return (np.stack([-self.rho * self.Om * np.sin(ph), self.rho * self.Om * np.cos(ph), 0 * t], 1)
                + self.B * 2 * np.pi * self.g * np.cos(2 * np.pi * self.g * t[:, None] + self.ps))

    def a(self, t):
        ph = self.Om * t
        w2 = self.Om ** 2
        return (np.stack([-self.rho * w2 * np.cos(ph), -self.rho * w2 * np.sin(ph), 0 * t], 1)
                - self.B * (2 * np.pi * self.g) ** 2 * np.sin(2 * np.pi * self.g * t[:, None] + self.ps))

    def omega_body(self, t):
        E = _exp(self.theta(t))
        ez = _R0.T @ np.array([0.0, 0.0, 1.0])
        return (np.einsum("nji,j->ni", E, ez) * self.Om
                + np.einsum("nij,nj->ni", _jr(self.theta(t)), self.theta_dot(t)))


def _preintegrate_batch(gyro, accel, dt, bhat, gyro_nd, accel_nd, gyro_rw, accel_rw):
    """Midpoint preintegration with bias Jacobians and covariance, batched over
    keyframe pairs (the scheme of imu.py:77-167).  gyro/accel: [F, S+1, 3]."""
    F, S1, _ = gyro.shape
    gyro = gyro - bhat[:, None, 0:3]
    accel = accel - bhat[:, None, 3:6]
    I3 = np.eye(3)
    dR = np.broadcast_to(I3, (F, 3, 3)).copy()
    dv = np.zeros((F, 3))
    dp = np.zeros((F, 3))
    Jr_ = np.zeros((F, 3, 3))
    Jv = np.zeros((F, 3, 6))
    Jp = np.zeros((F, 3, 6))
    cov = np.zeros((F, 9, 9))
    sg2, sa2 = gyro_nd ** 2, accel_nd ** 2
    for k in range(S1 - 1):
        w = 0.5 * (gyro[:, k] + gyro[:, k + 1])
        a = 0.5 * (accel[:, k] + accel[:, k + 1])
        Ef, Eh = _exp(w * dt), _exp(w * (0.5 * dt))
        Jf, Jh = _jr(w * dt), _jr(w * (0.5 * dt))
        Rm = dR @ Eh
        ai = np.einsum("fij,fj->fi", Rm, a)
        Ah = _hat(a)
        Jmid = np.swapaxes(Eh, 1, 2) @ Jr_ - 0.5 * dt * Jh
        RAJ = Rm @ Ah @ Jmid
        RAE = Rm @ Ah @ np.swapaxes(Eh, 1, 2)
        RAJh = Rm @ Ah @ Jh
        A = np.broadcast_to(np.eye(9), (F, 9, 9)).copy()
        A[:, 0:3, 0:3] = np.swapaxes(Ef, 1, 2)
        A[:, 3:6, 0:3] = -0.5 * dt * dt * RAE
        A[:, 3:6, 6:9] = dt * I3
        A[:, 6:9, 0:3] = -dt * RAE
        B = np.zeros((F, 9, 6))
        B[:, 0:3, 0:3] = -dt * Jf
        B[:, 3:6, 0:3] = 0.25 * dt ** 3 * RAJh
        B[:, 3:6, 3:6] = -0.5 * dt * dt * Rm
        B[:, 6:9, 0:3] = 0.5 * dt * dt * RAJh
        B[:, 6:9, 3:6] = -dt * Rm
        Qd = np.diag([sg2 / dt] * 3 + [sa2 / dt] * 3)
        cov = A @ cov @ np.swapaxes(A, 1, 2) + B @ Qd @ np.swapaxes(B, 1, 2)
        cov = 0.5 * (cov + np.swapaxes(cov, 1, 2))
        Jp[:, :, 0:3] += dt * Jv[:, :, 0:3] - 0.5 * dt * dt * RAJ
        Jp[:, :, 3:6] += dt * Jv[:, :, 3:6] - 0.5 * dt * dt * Rm
        Jv[:, :, 0:3] += -dt * RAJ
        Jv[:, :, 3:6] += -dt * Rm
        Jr_ = np.swapaxes(Ef, 1, 2) @ Jr_ - dt * Jf
        dp = dp + dv * dt + 0.5 * dt * dt * ai
        dv = dv + dt * ai
        dR = dR @ Ef
    dt_total = dt * (S1 - 1)
    C = np.zeros((F, 15, 15))
    C[:, :9, :9] = cov
    C[:, 9:12, 9:12] = gyro_rw ** 2 * dt_total * I3
    C[:, 12:15, 12:15] = accel_rw ** 2 * dt_total * I3
    return dR, dp, dv, Jr_, Jp, Jv, C


def _nearest_targets(i, K, deg):
    cand = sorted((abs(j - i), j) for j in range(K) if j != i)
    return [j for _, j in cand[:deg]]


def make_workload(cfg: int, grid=None, seed=None, with_truth=False):
    """Build the seeded FrameGraph for BASELINE config ``cfg``.

    ``grid`` overrides (rows, cols) for reduced fixtures.  Returns the graph,
    or (graph, truth_states) with ``with_truth``.
    """
    spec = CONFIGS[cfg]
    rows, cols = grid or spec.grid
    K = spec.n_kf
    rng = np.random.default_rng(1000 + cfg if seed is None else seed)
    mot = _Motion(rng)
    g_world = np.array([0.0, 0.0, GRAVITY])      # GravityModel.vector() with R_wg = I

    # --- IMU stream and true states (midpoint integration of the clean signal)
    n_s = (K - 1) * IMU_STEPS + 1
    dt = 1.0 / RATE
    ts = np.arange(n_s) * dt
    Rt = mot.R(ts)
    gyro_c = mot.omega_body(ts)
    acc_c = np.einsum("nji,nj->ni", Rt, mot.a(ts) - g_world)
    R = Rt[0].copy()
    p = mot.p(ts[:1])[0].copy()
    v = mot.v(ts[:1])[0].copy()
    states = [(R.copy(), p.copy(), v.copy())]
    for n in range(n_s - 1):
        w = 0.5 * (gyro_c[n] + gyro_c[n + 1])
        a = 0.5 * (acc_c[n] + acc_c[n + 1])
        Rm = R @ _exp(w * dt / 2.0)
        aw = Rm @ a + g_world
        p = p + v * dt + 0.5 * dt * dt * aw
        v = v + dt * aw
        R = R @ _exp(w * dt)
        if (n + 1) % IMU_STEPS == 0:
            states.append((R.copy(), p.copy(), v.copy()))

    gyro_nd = SIGMA_GYRO / np.sqrt(RATE)
    accel_nd = SIGMA_ACC / np.sqrt(RATE)
    g_rw, a_rw = 1e-5, 1e-4
    bw_g = np.cumsum(np.vstack([np.zeros(3), g_rw * np.sqrt(dt) * rng.standard_normal((n_s - 1, 3))]), 0)
    bw_a = np.cumsum(np.vstack([np.zeros(3), a_rw * np.sqrt(dt) * rng.standard_normal((n_s - 1, 3))]), 0)
    b0 = np.concatenate([rng.normal(0, 2e-3, 3), rng.normal(0, 2e-2, 3)])
    bias_t = np.hstack([bw_g, bw_a]) + b0
    gyro_m = gyro_c + bias_t[:, 0:3] + SIGMA_GYRO * rng.standard_normal((n_s, 3))
    acc_m = acc_c + bias_t[:, 3:6] + SIGMA_ACC * rng.standard_normal((n_s, 3))
    b_true = bias_t[::IMU_STEPS]
    b_hat = b_true + rng.normal(0.0, 1e-3, b_true.shape)

    idx = np.arange(K - 1)[:, None] * IMU_STEPS + np.arange(IMU_STEPS + 1)[None, :]
    dR, dP, dV, JR, JP, JV, COV = _preintegrate_batch(
        gyro_m[idx], acc_m[idx], dt, b_hat[:-1], gyro_nd, accel_nd, g_rw, a_rw)

    # --- intrinsics and per-keyframe disparity grids
    s = spec.intr_scale
    # BASELINE: "fx=fy=320, cx=32, cy=24 at 1/8 resolution" — fx=320 is the
    # full-resolution (512x384) focal length, so the 1/8 grid uses fx=40
    # (77° FOV); cx, cy are already 1/8-resolution values.  DESIGN.md §7.
    fx = fy = FX_FULL / 8.0 * s
    cx, cy = 32.0 * s, 24.0 * s
    W = max(cols, int(np.ceil(cx)) + 1)
    Hh = max(rows, int(np.ceil(cy)) + 1)
    intr = T.Intrinsics(fx, fy, cx, cy, W, Hh)
    vv, uu = np.meshgrid(np.arange(rows, dtype=float), np.arange(cols, dtype=float), indexing="ij")
    pix = np.stack([uu.ravel(), vv.ravel()], 1)
    N = len(pix)
    depth = rng.uniform(0.5, 5.0, (K, N)).astype(np.float32).astype(float)
    disp_true = (1.0 / depth).astype(np.float32).astype(float)
    ray = np.stack([(pix[:, 0] - cx) / fx, (pix[:, 1] - cy) / fy, np.ones(N)], 1)

    # --- edges
    L = spec.n_loop
    base, extra = divmod(spec.n_edges - L, K)
    pairs = []
    for i in range(K):
        deg = min(K - 1, base + (1 if i < extra else 0))
        pairs += [(i, j) for j in _nearest_targets(i, K, deg)]
    if L:
        cand = []
        for i in range(K):
            for j in range(K):
                if abs(i - j) <= 30:
                    continue
                Ri, pi_, _ = states[i]
                Rj, pj, _ = states[j]
                ang = np.linalg.norm(_log(Ri.T @ Rj))
                if np.linalg.norm(pi_ - pj) <= 0.3 and ang <= np.deg2rad(15.0):
                    cand.append((i, j))
        if len(cand) < L:
            raise RuntimeError(f"only {len(cand)} covisible loop candidates for {L} loop edges")
        pick = rng.choice(len(cand), size=L, replace=False)
        pairs += [cand[k] for k in sorted(pick)]
    pairs.sort(key=lambda ij: (ij[0], ij[1]))

    edges = []
    for (i, j) in pairs:
        Ri, pi_, _ = states[i]
        Rj, pj, _ = states[j]
        Xw = (ray / disp_true[i][:, None]) @ Ri.T + pi_
        Xj = (Xw - pj) @ Rj
        z = Xj[:, 2]
        zs = np.where(z > 0.05, z, 1.0)
        uv = np.stack([fx * Xj[:, 0] / zs + cx, fy * Xj[:, 1] / zs + cy], 1)
        # reference provider visibility rule (synth.py:553-556): in front and inside the image
        ok = ((z > 0.05) & (uv[:, 0] >= 0.0) & (uv[:, 0] <= W - 1.0)
              & (uv[:, 1] >= 0.0) & (uv[:, 1] <= Hh - 1.0))
        tgt = uv + spec.sigma_px * rng.standard_normal((N, 2))
        w = rng.uniform(0.0, 1.0, (N, 2))
        if spec.outlier_rate > 0:
            bad = rng.random(N) < spec.outlier_rate
            tgt[bad] += rng.uniform(-20.0, 20.0, (int(bad.sum()), 2))
            w[bad] = 0.05
        tgt = np.where(ok[:, None], tgt, pix)
        w[~ok] = 0.0
        edges.append(T.VisionEdge(i, j, pix, tgt.astype(np.float32).astype(float),
                                  w.astype(np.float32).astype(float)))

    # --- keyframes (initial estimate = perturbed truth)
    kfs = []
    truth = []
    for n in range(K):
        Rn, pn, vn = states[n]
        st = T.PoseState(T.Pose(T.Rotation.from_matrix(Rn), pn.copy()), vn.copy(),
                         T.BiasState(b_true[n, 0:3].copy(), b_true[n, 3:6].copy()), n * KF_DT)
        truth.append(st)
        if n == 0:
            est_pose, est_v = st.pose.copy(), vn.copy()
        else:
            ax = rng.standard_normal(3)
            ax /= np.linalg.norm(ax)
            dpv = rng.standard_normal(3)
            dpv *= 0.05 / np.linalg.norm(dpv)
            est_pose = st.pose.retract(ax * np.deg2rad(2.0), dpv)
            est_v = vn + rng.standard_normal(3) * 0.02
        bias = T.BiasState(b_hat[n, 0:3].copy(), b_hat[n, 3:6].copy())
        d0 = (disp_true[n] * rng.uniform(0.97, 1.03, N)).astype(np.float32).astype(float)
        kfs.append(T.Keyframe(n, T.PoseState(est_pose, est_v, bias, n * KF_DT), pix, d0))

    imu = []
    for f in range(K - 1):
        imu.append((f, f + 1, T.PreintegratedDelta(
            dt_total=IMU_STEPS * dt, delta_R=T.Rotation.from_matrix(dR[f]), delta_p=dP[f],
            delta_v=dV[f], J_rot=JR[f], J_pos=JP[f], J_vel=JV[f], covariance=COV[f],
            bias_lin_point=T.BiasState(b_hat[f, 0:3].copy(), b_hat[f, 3:6].copy()))))

    graph = T.FrameGraph(kfs, edges, imu, T.GravityModel(), intr)
    # the raw IMU stream the deltas were preintegrated from (pair f: samples idx[f])
    graph.imu_stream = {"ts": ts, "gyro": gyro_m, "accel": acc_m, "idx": idx, "bias": b_hat[:-1].copy(),
                        "noise": (gyro_nd, accel_nd, g_rw, a_rw)}
    return (graph, truth) if with_truth else graph


def _log(R):
    return T.Rotation.from_matrix(R).log()


def workload_stats(graph) -> dict:
    E = len(graph.vision_edges)
    N = len(graph.keyframes[0].disparities) if graph.keyframes else 0
    rows = sum(len(e.pixels) for e in graph.vision_edges)
    return {"n_kf": len(graph.keyframes), "n_edges": E, "px_per_kf": N, "edge_px": rows}


# --------------------------------------------------------------------------
# Pose-graph (PGBA) stress window: SURVEY.md §8(f)#1.  Not a BASELINE config (the
# reference publishes none for PGBA); shaped like the paper's loop closure over a
# long drifting trajectory: K keyframes on 1.25 laps of a 2 m circle (revisits after
# one lap), Sim(3) odometry with a creeping scale drift as the chain, and loop edges
# between revisiting keyframes carrying dense 48x64 correspondences (BASELINE
# intrinsics) plus the exact relative pose.
# --------------------------------------------------------------------------

CHAIN_INFO = np.diag([4e4] * 3 + [1e4] * 3 + [100.0])   # test_loopclosure.py:38


def _sim3(R, t, s=1.0):
    return T.SimTransform(T.Rotation.from_matrix(R), np.asarray(t, float), s)


def make_pgba_workload(n_nodes=256, n_loops=8, grid=(48, 64), seed=2024, drift=1.05, sigma_px=0.5):
    """Seeded PoseGraph (paper_2512_02293_b200.types) + the true node states."""
    rng = np.random.default_rng(seed)
    rows, cols = grid
    lap = int(round(n_nodes / 1.25))
    ang = 2.0 * np.pi * np.arange(n_nodes) / lap
    gt = []
    for a in ang:
        p = np.array([2.0 * np.cos(a), 2.0 * np.sin(a), 0.1 * np.sin(3.0 * a)])
        # camera looks outward from the circle (z axis radial), yaw follows the angle
        Rz = _rz(a)
        R = Rz @ np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
        gt.append(_sim3(R, p))
    sig = drift ** (1.0 / (n_nodes - 1))
    odo = [gt[0].copy()]
    chain = []
    for k in range(n_nodes - 1):
        rel = gt[k + 1] * gt[k].inverse()
        noise = T.Rotation.exp(rng.normal(0.0, 2e-4, 3))
        meas = T.SimTransform(rel.rotation * noise, rel.translation + rng.normal(0.0, 5e-4, 3), sig)
        odo.append(meas * odo[k])
        chain.append(T.RelativePoseEdge(k, k + 1, meas, CHAIN_INFO))
    fx = fy = FX_FULL / 8.0
    cx, cy = 32.0, 24.0
    intr = T.Intrinsics(fx, fy, cx, cy, max(cols, 33), max(rows, 25))
    vv, uu = np.meshgrid(np.arange(rows, dtype=float), np.arange(cols, dtype=float), indexing="ij")
    pix = np.stack([uu.ravel(), vv.ravel()], 1)
    N = len(pix)
    ray = np.stack([(pix[:, 0] - cx) / fx, (pix[:, 1] - cy) / fy, np.ones(N)], 1)
    # loop pairs: j revisits i one lap later
    cand = np.arange(0, n_nodes - lap)
    srcs = np.sort(rng.choice(cand, size=min(n_loops, len(cand)), replace=False))
    nodes = [T.PoseGraphNode(k, odo[k].copy(), timestamp=float(k) * KF_DT) for k in range(n_nodes)]
    loops = []
    for i in srcs:
        j = int(i + lap)
        depth = rng.uniform(0.5, 5.0, N).astype(np.float32).astype(float)
        d_true = (1.0 / depth).astype(np.float32).astype(float)
        Xw = gt[i].apply(ray / d_true[:, None])
        Xj = gt[j].inverse().apply(Xw)
        z = Xj[:, 2]
        zs = np.where(z > 0.05, z, 1.0)
        uv = np.stack([fx * Xj[:, 0] / zs + cx, fy * Xj[:, 1] / zs + cy], 1)
        ok = (z > 0.05) & (uv[:, 0] >= 0) & (uv[:, 0] <= cols - 1) & (uv[:, 1] >= 0) & (uv[:, 1] <= rows - 1)
        tgt = np.where(ok[:, None], uv + sigma_px * rng.standard_normal((N, 2)), pix)
        w = rng.uniform(0.0, 1.0, (N, 2))
        w[~ok] = 0.0
        nodes[i].pixels = pix.copy()
        nodes[i].disparities = (d_true * rng.uniform(0.97, 1.03, N)).astype(np.float32).astype(float)
        rel = T.RelativePoseEdge(int(i), j, gt[j] * gt[i].inverse(), np.eye(7) * 1e6)
        vis = T.VisionEdge(int(i), j, pix.copy(), tgt.astype(np.float32).astype(float),
                           w.astype(np.float32).astype(float))
        loops.append(T.LoopEdge(int(i), j, rel, vis))
    graph = T.PoseGraph(nodes, chain, loops, intr, None, min_loop_gap=55)
    return graph, gt
