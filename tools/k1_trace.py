"""Tuning: fraction of K1 warp time spent waiting for streamed stages (VBA_K1_TRACE builds)."""
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
dp = DeviceProblem(P, {"max_iterations": CONFIGS[cfg].iterations})
lib = ctypes.CDLL(os.environ["VBA_LIB"])
buf = (ctypes.c_ulonglong * 4)()
dp.linearize()
lib.vba_k1_trace(buf)
for _ in range(3):
    dp.linearize()
lib.vba_k1_trace(buf)
w, t, n = buf[0], buf[1], buf[2]
print(f"cfg{cfg}: warp-items {n}, wait {w / max(t, 1) * 100:.1f}% of warp cycles, "
      f"{t / max(n, 1):.0f} cyc/warp-item total, {w / max(n, 1):.0f} waiting, "
      f"skipped pixel blocks {buf[3] / max(4 * n, 1) * 100:.1f}%")

ends = (ctypes.c_ulonglong * 1024)()
dp.linearize()
lib.vba_k1_ends(ends)
e = sorted(x for x in ends if x)
if e:
    import statistics
    print(f"CTA finish spread: first {0:.1f} us, median {(statistics.median(e) - e[0]) / 1e3:.1f} us, "
          f"p90 {(e[int(0.9 * len(e))] - e[0]) / 1e3:.1f} us, last {(e[-1] - e[0]) / 1e3:.1f} us over {len(e)} CTAs")
