"""Time the native LM solve on BASELINE configs 0-4 (device-resident inputs) with a stage breakdown."""
import argparse
import os
import sys
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2512_02293_b200.device import DeviceProblem  # noqa: E402
from paper_2512_02293_b200.problem import pack_graph  # noqa: E402
from paper_2512_02293_b200.workloads import CONFIGS, make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2,3,4")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

for cfg in [int(c) for c in a.configs.split(",")]:
    t0 = time.time()
    g = make_workload(cfg)
    P = pack_graph(g)
    spec = CONFIGS[cfg]
    dp = DeviceProblem(P, {"max_iterations": spec.iterations})
    tprep = time.time() - t0
    edge_px = int(sum(len(e.pixels) for e in g.vision_edges))
    for _ in range(2):
        dp.load_state()
        rep = dp.solve()
    dp.set_profiling(True)
    dp.load_state()
    rep = dp.solve()
    st = dp.stage_times()
    dp.set_profiling(False)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(a.reps):
        dp.load_state()
        torch.cuda.synchronize()
        ev0.record(dp.stream)
        rep = dp.solve()
        ev1.record(dp.stream)
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    ms = min(ts)
    it = rep["iterations"]
    print(f"cfg{cfg}: K={spec.n_kf} E={len(g.vision_edges)} edge_px={edge_px} nfree={dp.lib.vba_reduced_dim(dp.ctx)} "
          f"prep {tprep:.1f}s | solve {ms:.2f} ms, it={it} trials={rep['trials']} term={rep['termination']} "
          f"| {edge_px * it / ms * 1e3:.3e} edge-px/s, {it / ms * 1e3:.1f} it/s")
    print("   stages(ms): " + " ".join(f"{k}={v:.3f}" for k, v in st.items()))
    print("   costs: " + " ".join(f"{c:.4e}" for c in rep["cost_trajectory"]))
    import ctypes
    stt = (ctypes.c_int64 * 4)()
    dp.lib.vba_stats(dp.ctx, stt)
    print(f"   tensor-core solve: {bool(stt[0])}, fp64 fallbacks {stt[1]}, solves {stt[2]}, "
          f"refinement passes/solve {stt[3] / max(stt[2], 1):.1f}")
    dp.close()
    del dp
    torch.cuda.empty_cache()
