"""Diagnostics: timeline of DeviceProblem.solve_windows (uploads on the copy stream vs solves)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02293_b200.device import DeviceProblem  # noqa: E402
from paper_2512_02293_b200.problem import pack_graph  # noqa: E402
from paper_2512_02293_b200.workloads import CONFIGS, make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
P = pack_graph(make_workload(cfg))
dp = DeviceProblem(P, {"max_iterations": CONFIGS[cfg].iterations})
H = dp.H
pinned = {k: torch.from_numpy(np.ascontiguousarray(v).reshape(-1)).pin_memory()
          for k, v in (("state", H.state), ("disp64", H.disp64), ("tgt", H.tgt), ("w", H.w), ("imu", H.imu),
                       ("grav", H.grav))}
dp.solve_windows([pinned])
torch.cuda.synchronize()
# plain H2D bandwidth of the two big arrays
t = torch.empty_like(dp.d_tgt)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t.copy_(pinned["tgt"], non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"H2D tgt {pinned['tgt'].numel() * 4 / 1e6:.0f} MB: {e0.elapsed_time(e1):.2f} ms")
# solve alone
e0.record(dp.stream)
dp.load_state()
dp.solve()
e1.record(dp.stream)
torch.cuda.synchronize()
print(f"solve alone {e0.elapsed_time(e1):.2f} ms")
h0 = time.perf_counter()
e0.record(dp.stream)
dp.solve_windows([pinned] * K)
e1.record(dp.stream)
torch.cuda.synchronize()
print(f"solve_windows x{K}: {e0.elapsed_time(e1):.2f} ms device, {1e3 * (time.perf_counter() - h0):.2f} ms host")

# explicit timeline of the same schedule
from paper_2512_02293_b200 import _lib as L  # noqa: E402
st = dp.stream
cs = torch.cuda.Stream(dp.device)
sets = ((dp.d_tgt, dp.d_w), dp._stage)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
base = ev()
base.record(st)
cs.wait_stream(st)
marks = []
up = [None, None]
free = [None, None]


def upload(b):
    with torch.cuda.stream(cs):
        if free[b] is not None:
            cs.wait_event(free[b])
        a0 = ev(); a0.record(cs)
        sets[b][0].copy_(pinned["tgt"], non_blocking=True)
        sets[b][1].copy_(pinned["w"], non_blocking=True)
        a1 = ev(); a1.record(cs)
        up[b] = a1
        return a0, a1


ups = [upload(0)]
for s in range(K):
    b = s & 1
    if s + 1 < K:
        ups.append(upload(b ^ 1))
    st.wait_event(up[b])
    s0 = ev(); s0.record(st)
    L.check(dp.lib.vba_bind_inputs(dp.ctx, dp._sptr(), sets[b][0].data_ptr(), sets[b][1].data_ptr(), 1))
    dp.load_state()
    dp.solve()
    s1 = ev(); s1.record(st)
    free[b] = ev(); free[b].record(st)
    marks.append((s0, s1))
torch.cuda.synchronize()
for s in range(K):
    a0, a1 = ups[s]
    s0, s1 = marks[s]
    print(f"window {s}: upload {base.elapsed_time(a0):7.1f} -> {base.elapsed_time(a1):7.1f} | "
          f"solve {base.elapsed_time(s0):7.1f} -> {base.elapsed_time(s1):7.1f}")
