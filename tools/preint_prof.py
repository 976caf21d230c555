"""Times the batched IMU preintegration kernel (vba_preintegrate) on a synthetic window
and the CPU oracle on a bounded sample of it.  Prints one JSON line.

    python tools/preint_prof.py [--pairs 256] [--samples 200]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02293_b200 import _lib  # noqa: E402
from paper_2512_02293_b200.imu import preintegrate_device, scratch_for, unpack  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=256)
    ap.add_argument("--samples", type=int, default=200)   # 200 Hz IMU, 1 s between keyframes
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    rng = np.random.default_rng(7)
    F, S = a.pairs, a.samples
    ts = np.concatenate([f * 1.0 + np.arange(S) / 200.0 + rng.uniform(0, 1e-4, S) for f in range(F)])
    gyro = rng.normal(0, 0.5, (F * S, 3))
    accel = rng.normal(0, 1.0, (F * S, 3)) + np.array([0, 0, 9.81])
    soff = np.arange(F + 1, dtype=np.int64) * S
    bias = rng.normal(0, 1e-3, (F, 6))
    noise = np.array([1.7e-4, 2e-3, 1e-5, 1e-4])
    dev = [torch.from_numpy(x).cuda() for x in (ts, gyro, accel, soff, bias, noise)]
    out = torch.empty((F, _lib.PREINT_REC), dtype=torch.float64, device="cuda")
    ws = scratch_for(F * S)
    for _ in range(3):
        preintegrate_device(*dev, out=out, scratch=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        preintegrate_device(*dev, out=out, scratch=ws)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1) / a.reps
    res = unpack(out.cpu().numpy())
    from oracle.imu import preintegrate as oracle_preintegrate
    n_cpu = max(1, min(F, 8))
    t0 = time.perf_counter()
    worst = 0.0
    for f in range(n_cpu):
        sl = slice(f * S, (f + 1) * S)
        d = oracle_preintegrate(ts[sl], gyro[sl], accel[sl], bias[f], noise)
        for k in ("delta_q", "delta_p", "delta_v", "J_rot", "J_pos", "J_vel", "covariance"):
            worst = max(worst, float(np.abs(res[k][f] - d[k]).max() / max(np.abs(d[k]).max(), 1e-300)))
    cpu_s = (time.perf_counter() - t0) / n_cpu
    print(json.dumps({"pairs": F, "samples_per_pair": S, "gpu_ms_per_window": gpu_ms,
                      "gpu_intervals_per_s": F * (S - 1) / (gpu_ms * 1e-3),
                      "cpu_oracle_s_per_pair": cpu_s, "cpu_intervals_per_s": (S - 1) / cpu_s,
                      "max_rel_diff_vs_oracle": worst}))


if __name__ == "__main__":
    main()
