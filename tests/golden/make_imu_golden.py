"""Golden vectors for IMU preintegration from the REFERENCE (build container only).

Runs vislam.imu.preintegrate (imu.py:77-167) on seeded sample streams — 200 Hz
samples between 10 Hz keyframes as BASELINE.json's configs, plus edge cases: two
samples, a near-zero rotation (small-angle branches of geometry.py) and a fast
rotation (non-positive trace branch of Rotation.from_matrix) — and writes
tests/golden/imu/imu_preint.npz.  Run:  python tests/golden/make_imu_golden.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from vislam.imu import BiasState, ImuNoiseModel, ImuSample, preintegrate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(2512)
noise = ImuNoiseModel(gyro_noise_density=0.002 / np.sqrt(200), accel_noise_density=0.02 / np.sqrt(200),
                      gyro_bias_random_walk=1e-5, accel_bias_random_walk=1e-4)
cases = []
for c in range(12):
    S = 2 if c == 0 else int(rng.integers(5, 24))
    t0 = float(rng.uniform(0, 10))
    dts = rng.uniform(0.004, 0.006, S - 1)
    ts = t0 + np.concatenate([[0.0], np.cumsum(dts)])
    scale = 1e-10 if c == 1 else (40.0 if c == 2 else 1.0)   # tiny / fast rotation
    gyro = scale * rng.normal(0, 0.8, (S, 3))
    accel = rng.normal(0, 1.0, (S, 3)) + np.array([0.0, 0.0, 9.81])
    bias = np.concatenate([rng.normal(0, 2e-3, 3), rng.normal(0, 2e-2, 3)])
    samples = [ImuSample(float(ts[k]), gyro[k], accel[k]) for k in range(S)]
    d = preintegrate(samples, BiasState(bias[:3], bias[3:]), noise)
    cases.append(dict(ts=ts, gyro=gyro, accel=accel, bias=bias, dt_total=d.dt_total, delta_q=d.delta_R.q,
                      delta_p=d.delta_p, delta_v=d.delta_v, J_rot=d.J_rot, J_pos=d.J_pos, J_vel=d.J_vel,
                      covariance=d.covariance))
out = {"noise": np.array([noise.gyro_noise_density, noise.accel_noise_density, noise.gyro_bias_random_walk,
                          noise.accel_bias_random_walk]), "n": np.array(len(cases))}
for i, cs in enumerate(cases):
    for k, v in cs.items():
        out[f"c{i}_{k}"] = np.asarray(v, float)
np.savez_compressed(os.path.join(HERE, "imu", "imu_preint.npz"), **out)
print("wrote", len(cases), "cases")
