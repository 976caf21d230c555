"""Host-side data types mirroring the reference solver's interface.

Field names and validation follow the reference dataclasses so that graphs
built with either package are interchangeable (the B200 solver reads them
duck-typed):

* ``Keyframe``, ``FrameGraph``, ``SolveOptions``, ``SolveReport``
  — /root/reference/pkg/src/vislam/solver.py:37-115
* ``PoseState``, ``Intrinsics``, ``VisionEdge``, ``GravityModel``
  — residuals.py:34-137
* ``BiasState``, ``PreintegratedDelta`` — imu.py:29-74
* ``Rotation``, ``Pose`` — geometry.py:101-229 (quaternion wxyz, w >= 0)

These are plain containers; all solver arithmetic runs on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_SMALL_ANGLE = 1e-8


def _qmul(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def _canon(q):
    q = np.asarray(q, dtype=float)
    q = q / np.linalg.norm(q)
    return -q if q[0] < 0.0 else q


class Rotation:
    """Unit quaternion (w, x, y, z), canonical w >= 0."""

    __slots__ = ("q",)

    def __init__(self, q):
        self.q = _canon(q)

    @staticmethod
    def identity():
        return Rotation(np.array([1.0, 0.0, 0.0, 0.0]))

    @staticmethod
    def exp(omega):
        omega = np.asarray(omega, dtype=float)
        th = float(np.linalg.norm(omega))
        if th < _SMALL_ANGLE:
            return Rotation(np.concatenate(([1.0], 0.5 * omega)))
        return Rotation(np.concatenate(([np.cos(0.5 * th)], np.sin(0.5 * th) * omega / th)))

    @staticmethod
    def from_matrix(R):
        R = np.asarray(R, dtype=float)
        t = np.trace(R)
        if t > 0.0:
            s = np.sqrt(t + 1.0) * 2.0
            q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
        else:
            i = int(np.argmax(np.diag(R)))
            a, b, c = i, (i + 1) % 3, (i + 2) % 3
            s = np.sqrt(1.0 + R[a, a] - R[b, b] - R[c, c]) * 2.0
            q = [0.0] * 4
            q[0] = (R[c, b] - R[b, c]) / s
            q[1 + a] = 0.25 * s
            q[1 + b] = (R[a, b] + R[b, a]) / s
            q[1 + c] = (R[a, c] + R[c, a]) / s
        return Rotation(np.array(q))

    def matrix(self):
        w, x, y, z = self.q
        return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                         [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                         [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])

    def log(self):
        w, v = self.q[0], self.q[1:]
        n = float(np.linalg.norm(v))
        if n < _SMALL_ANGLE:
            return (2.0 / w) * v
        return (2.0 * np.arctan2(n, w) / n) * v

    def inverse(self):
        w, x, y, z = self.q
        return Rotation(np.array([w, -x, -y, -z]))

    def apply(self, v):
        return np.asarray(v, dtype=float) @ self.matrix().T

    def __mul__(self, other):
        return Rotation(_qmul(self.q, other.q))

    def angle_to(self, other):
        return float(np.linalg.norm((self.inverse() * other).log()))

    def __repr__(self):
        return f"Rotation(q={self.q})"


@dataclass
class Pose:
    rotation: Rotation
    translation: np.ndarray

    def __post_init__(self):
        self.translation = np.asarray(self.translation, dtype=float).reshape(3)

    @staticmethod
    def identity():
        return Pose(Rotation.identity(), np.zeros(3))

    def apply(self, x):
        return self.rotation.apply(x) + self.translation

    def compose(self, other):
        return Pose(self.rotation * other.rotation,
                    self.rotation.apply(other.translation) + self.translation)

    __mul__ = compose

    def inverse(self):
        ri = self.rotation.inverse()
        return Pose(ri, -ri.apply(self.translation))

    def retract(self, dtheta, dp):
        return Pose(self.rotation * Rotation.exp(dtheta), self.translation + dp)

    def copy(self):
        return Pose(Rotation(self.rotation.q.copy()), self.translation.copy())


@dataclass
class BiasState:
    gyro_bias: np.ndarray = field(default_factory=lambda: np.zeros(3))
    accel_bias: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.gyro_bias = np.asarray(self.gyro_bias, dtype=float).reshape(3)
        self.accel_bias = np.asarray(self.accel_bias, dtype=float).reshape(3)
        if not (np.all(np.isfinite(self.gyro_bias)) and np.all(np.isfinite(self.accel_bias))):
            raise ValueError("bias must be finite")

    def vector(self):
        return np.concatenate([self.gyro_bias, self.accel_bias])

    def copy(self):
        return BiasState(self.gyro_bias.copy(), self.accel_bias.copy())


@dataclass
class PreintegratedDelta:
    dt_total: float
    delta_R: Rotation
    delta_p: np.ndarray
    delta_v: np.ndarray
    J_rot: np.ndarray
    J_pos: np.ndarray
    J_vel: np.ndarray
    covariance: np.ndarray
    bias_lin_point: BiasState


@dataclass
class PoseState:
    pose: Pose
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    bias: BiasState = field(default_factory=BiasState)
    timestamp: float = 0.0

    def __post_init__(self):
        self.velocity = np.asarray(self.velocity, dtype=float).reshape(3)

    def copy(self):
        return PoseState(self.pose.copy(), self.velocity.copy(), self.bias.copy(), self.timestamp)


@dataclass
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError("focal lengths must be positive")
        if not (0.0 <= self.cx < self.width and 0.0 <= self.cy < self.height):
            raise ValueError("principal point must lie inside the image")


@dataclass
class VisionEdge:
    i: int
    j: int
    pixels: np.ndarray
    targets: np.ndarray
    weights: np.ndarray

    def __post_init__(self):
        self.pixels = np.asarray(self.pixels, dtype=float).reshape(-1, 2)
        self.targets = np.asarray(self.targets, dtype=float).reshape(-1, 2)
        self.weights = np.asarray(self.weights, dtype=float).reshape(-1, 2)
        n = len(self.pixels)
        if len(self.targets) != n or len(self.weights) != n:
            raise ValueError("pixels, targets and weights must have equal length")
        if np.any(self.weights < 0.0):
            raise ValueError("weights must be non-negative")


@dataclass
class GravityModel:
    R_wg: Rotation = field(default_factory=Rotation.identity)
    magnitude: float = 9.81

    def __post_init__(self):
        if not self.magnitude > 0.0:
            raise ValueError("gravity magnitude must be positive")

    def copy(self):
        return GravityModel(Rotation(self.R_wg.q.copy()), self.magnitude)


@dataclass
class Keyframe:
    kid: int
    state: PoseState
    pixels: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))
    disparities: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def __post_init__(self):
        self.pixels = np.asarray(self.pixels, dtype=float).reshape(-1, 2)
        self.disparities = np.asarray(self.disparities, dtype=float).reshape(-1)
        if len(self.pixels) != len(self.disparities):
            raise ValueError("one disparity per tracked pixel")
        if len(self.disparities) and self.disparities.min() <= 0.0:
            raise ValueError("disparities must be positive")


@dataclass
class FrameGraph:
    keyframes: list
    vision_edges: list
    inertial_edges: list
    gravity: GravityModel
    intrinsics: Intrinsics
    T_cb: Pose | None = None

    def __post_init__(self):
        ids = [kf.kid for kf in self.keyframes]
        if len(set(ids)) != len(ids):
            raise ValueError("duplicate keyframe ids")
        self._index = {kid: n for n, kid in enumerate(ids)}
        for e in self.vision_edges:
            if e.i not in self._index or e.j not in self._index:
                raise ValueError(f"vision edge ({e.i},{e.j}) references unknown keyframe")
        consecutive = {(ids[n], ids[n + 1]) for n in range(len(ids) - 1)}
        covered = {(i, j) for i, j, _ in self.inertial_edges}
        if self.inertial_edges and covered != consecutive:
            raise ValueError("inertial edges must cover exactly the consecutive pairs")

    def kf(self, kid):
        return self.keyframes[self._index[kid]]

    def index_of(self, kid):
        return self._index[kid]


@dataclass
class SolveOptions:
    max_iterations: int = 10
    damping: float = 1e-4
    damping_up: float = 10.0
    damping_down: float = 0.5
    rel_decrease_tol: float = 1e-8
    step_tol: float = 1e-10
    max_damping: float = 1e8
    frozen_keyframes: tuple = (0,)
    optimize_gravity: bool = False
    optimize_velocity_bias: bool = True
    use_schur: bool = True
    ridge: float = 1e-10

    def __post_init__(self):
        if self.max_iterations < 0:
            raise ValueError("max_iterations must be >= 0")
        for name in ("damping", "damping_up", "rel_decrease_tol", "step_tol",
                     "max_damping", "ridge"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if not (0 < self.damping_down < 1):
            raise ValueError("damping_down must be in (0, 1)")


@dataclass
class SolveReport:
    iterations: int
    initial_cost: float
    final_cost: float
    cost_trajectory: list
    termination: str
    condition_warnings: list = field(default_factory=list)


# ---------------------------------------------------------------------------
# Pose-graph (PGBA) containers: geometry.py:266-341 (SimTransform),
# residuals.py:144-156 (RelativePoseEdge), loopclosure.py:94-207 (LoopEdge,
# PoseGraphNode, PoseGraph, CorrectionEntry, LoopCorrection).  Containers only:
# SimTransform carries the host-side maps the drop-in needs for write-back and
# the correction message (compose / inverse / pose); the solve itself is on the GPU.
# ---------------------------------------------------------------------------

@dataclass
class SimTransform:
    """Similarity transform x_out = scale * R @ x + t, scale > 0."""

    rotation: Rotation
    translation: np.ndarray
    scale: float = 1.0

    def __post_init__(self):
        self.translation = np.asarray(self.translation, dtype=float).reshape(3)
        self.scale = float(self.scale)
        if not self.scale > 0.0:
            raise ValueError(f"scale must be positive, got {self.scale}")

    @staticmethod
    def identity():
        return SimTransform(Rotation.identity(), np.zeros(3), 1.0)

    @staticmethod
    def from_pose(pose, scale=1.0):
        return SimTransform(Rotation(pose.rotation.q.copy()), pose.translation.copy(), scale)

    def pose(self):
        return Pose(Rotation(self.rotation.q.copy()), self.translation.copy())

    def apply(self, x):
        return self.scale * self.rotation.apply(x) + self.translation

    def compose(self, other):
        return SimTransform(self.rotation * other.rotation,
                            self.scale * self.rotation.apply(other.translation) + self.translation,
                            self.scale * other.scale)

    __mul__ = compose

    def inverse(self):
        Rinv = self.rotation.inverse()
        inv_s = 1.0 / self.scale
        return SimTransform(Rinv, -inv_s * Rinv.apply(self.translation), inv_s)

    def copy(self):
        return SimTransform(Rotation(self.rotation.q.copy()), self.translation.copy(), self.scale)


@dataclass
class RelativePoseEdge:
    i: int
    j: int
    measurement: SimTransform
    information: np.ndarray

    def __post_init__(self):
        self.information = np.asarray(self.information, dtype=float).reshape(7, 7)
        if np.max(np.abs(self.information - self.information.T)) > 1e-9:
            raise ValueError("information must be symmetric")
        if np.linalg.eigvalsh(self.information).min() < -1e-9:
            raise ValueError("information must be PSD")


@dataclass
class LoopEdge:
    i: int
    j: int
    relative: RelativePoseEdge
    vision: VisionEdge | None = None

    def __post_init__(self):
        if not self.i < self.j:
            raise ValueError("loop endpoints must satisfy i < j")
        if (self.relative.i, self.relative.j) != (self.i, self.j):
            raise ValueError("relative edge endpoints must match the loop pair")
        if self.vision is not None and (self.vision.i, self.vision.j) != (self.i, self.j):
            raise ValueError("vision edge endpoints must match the loop pair")


@dataclass
class PoseGraphNode:
    kid: int
    state: SimTransform
    pixels: np.ndarray | None = None
    disparities: np.ndarray | None = None
    timestamp: float = 0.0


@dataclass
class PoseGraph:
    nodes: list
    chain: list
    loops: list
    intrinsics: Intrinsics | None = None
    T_cb: Pose | None = None
    min_loop_gap: int = 55

    def __post_init__(self):
        self.nodes = sorted(self.nodes, key=lambda n: n.kid)
        kids = [n.kid for n in self.nodes]
        if len(set(kids)) != len(kids):
            raise ValueError("duplicate pose graph node ids")
        self._index = {kid: n for n, kid in enumerate(kids)}
        consecutive = {(kids[n], kids[n + 1]) for n in range(len(kids) - 1)}
        covered = {(e.i, e.j) for e in self.chain}
        if self.chain and covered != consecutive:
            raise ValueError("chain must cover exactly the consecutive keyframe pairs")
        for loop in self.loops:
            if loop.i not in self._index or loop.j not in self._index:
                raise ValueError(f"loop edge ({loop.i},{loop.j}) references unknown keyframe")
            if loop.j - loop.i < self.min_loop_gap:
                raise ValueError(f"loop edge ({loop.i},{loop.j}) violates the keyframe gap gate")
            if loop.vision is not None:
                if self.intrinsics is None:
                    raise ValueError("vision loop edges need intrinsics")
                src = self.node(loop.i)
                if src.pixels is None or src.disparities is None:
                    raise ValueError(f"keyframe {loop.i} has no pixel snapshot for its loop edge")
                if len(src.disparities) != len(loop.vision.pixels):
                    raise ValueError("loop vision rows must align with the source pixel snapshot")

    def node(self, kid):
        return self.nodes[self._index[kid]]

    def index_of(self, kid):
        return self._index[kid]


@dataclass
class CorrectionEntry:
    kid: int
    old_pose: Pose
    new_pose: Pose
    scale_change: float = 1.0

    def __post_init__(self):
        self.scale_change = float(self.scale_change)
        if not self.scale_change > 0.0:
            raise ValueError("scale change must be positive")

    def delta(self):
        new = SimTransform(Rotation(self.new_pose.rotation.q.copy()), self.new_pose.translation.copy(),
                           self.scale_change)
        return new * SimTransform.from_pose(self.old_pose).inverse()


@dataclass
class LoopCorrection:
    entries: dict
    timestamp: float = 0.0


# ---------------------------------------------------------------------------
# Staged initialisation containers: initialization.py:30-61 (InitConfig, InitResult)
# ---------------------------------------------------------------------------

@dataclass
class InitConfig:
    n_vis_init: int = 10
    n_iner_init: int = 20
    max_iterations_vision: int = 30
    max_iterations_inertial: int = 60
    max_iterations_joint: int = 15
    damping: float = 1e-4

    def __post_init__(self):
        if not 2 <= self.n_vis_init <= self.n_iner_init:
            raise ValueError("need n_iner_init >= n_vis_init >= 2")
        for name in ("max_iterations_vision", "max_iterations_inertial", "max_iterations_joint"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be at least 1")


@dataclass
class InitResult:
    gravity: GravityModel
    log_scale: float
    velocities: np.ndarray
    bias: BiasState
    reports: dict = field(default_factory=dict)

    def scale(self):
        return float(np.exp(self.log_scale))
