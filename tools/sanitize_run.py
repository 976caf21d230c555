"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck).

Runs every kernel family of libvba at sizes the sanitizers finish in minutes:
K1/K2/K3/K4/K6/K7 (linearise, energy, IMU, Schur Gram + fill transform, back-substitution,
retraction) through a 2-iteration solve of BASELINE config 1; the tensor-core reduced
solve (k_tc_diag/convert, k_chol_tc (PREP tasks), k_tc_fwd/bwd, k_tc_symv/resid, k_tc_check)
forced on that 2-tile system and on a standalone 8-tile SPD system; the fp64 tile-DAG
Cholesky; the dense (use_schur=False) path on a small golden window; IMU preintegration.
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_02293_b200 import _lib  # noqa: E402
from paper_2512_02293_b200.device import DeviceProblem  # noqa: E402
from paper_2512_02293_b200.problem import pack_graph  # noqa: E402
from paper_2512_02293_b200.workloads import make_workload  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
P = pack_graph(make_workload(1))
if which in ("all", "solve"):
    dp = DeviceProblem(P, {"max_iterations": 2})
    print("solve", dp.solve()["cost_trajectory"])
    dp.download()
    dp.close()
if which in ("all", "tc"):
    os.environ["VBA_CHOL"] = "tc"
    dp = DeviceProblem(P, {"max_iterations": 1})
    print("solve tc", dp.solve()["cost_trajectory"], dp.stats())
    dp.close()
    os.environ.pop("VBA_CHOL")
    n = 1000
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    H = A @ A.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    x0, tc = _lib.spd_solve(H, b, mode=0)
    x1, _ = _lib.spd_solve(H, b, mode=1)
    print("spd", tc, float((x0 - x1).abs().max()))
if which in ("all", "dense"):
    from conftest import load_golden
    Q, _, opts = load_golden("win6_frozen2")
    dp = DeviceProblem(Q, dict(opts, use_schur=False))
    dp.linearize()
    print("dense step", np.abs(dp.solve_step(1e-4, use_schur=False)[0]).max())
    dp.close()
if which in ("all", "preint"):
    from paper_2512_02293_b200 import imu
    s = make_workload(1).imu_stream
    idx = s["idx"]
    ts = [s["ts"][i] for i in idx]
    gy = [s["gyro"][i] for i in idx]
    ac = [s["accel"][i] for i in idx]
    d = imu.preintegrate_batch(ts, gy, ac, s["bias"], s["noise"])
    print("preint", d["delta_p"].shape)
torch.cuda.synchronize()
print("sanitize_run ok")
