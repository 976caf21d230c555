"""Tuning: per-warp cycle split of the Schur Gram kernel (VBA_GRAM_PROF builds, VBA_LIB=<variant>)."""
import ctypes
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2512_02293_b200.device import DeviceProblem  # noqa: E402
from paper_2512_02293_b200.problem import pack_graph  # noqa: E402
from paper_2512_02293_b200.workloads import CONFIGS, make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
P = pack_graph(make_workload(cfg))
dp = DeviceProblem(P, {"max_iterations": 1})
lib = ctypes.CDLL(os.environ["VBA_LIB"])
buf = (ctypes.c_ulonglong * 5)()
dp.solve()
lib.vba_gram_prof(buf)
dp.solve()
lib.vba_gram_prof(buf)
n = max(buf[4], 1)
tot = sum(buf[:4])
names = ["phase1 (coupling vectors)", "barrier after phase1", "phase2 (DMMA)", "barrier after phase2"]
print(f"cfg{cfg}: {n} warp-chunks, {tot / n:.0f} cycles per warp-chunk")
for i, nm in enumerate(names):
    print(f"  {nm:28s} {buf[i] / n:8.0f} cyc  {buf[i] / max(tot, 1) * 100:5.1f}%")
