import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2512_02293_b200.device import DeviceProblem
from paper_2512_02293_b200.problem import pack_graph
from paper_2512_02293_b200.workloads import CONFIGS, make_workload
P = pack_graph(make_workload(4))
dp = DeviceProblem(P, {"max_iterations": 2})
H = dp.H
pinned = {k: torch.from_numpy(np.ascontiguousarray(v).reshape(-1)).pin_memory()
          for k, v in (("state", H.state), ("disp64", H.disp64), ("tgt", H.tgt), ("w", H.w), ("imu", H.imu), ("grav", H.grav))}
outs = [(torch.empty(dp.d_state.shape, dtype=torch.float64).pin_memory(),
         torch.empty(dp.d_disp.shape, dtype=torch.float32).pin_memory()) for _ in range(10)]
dp.solve_windows([pinned], outputs=outs[:1]); torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dp.stream)
    dp.solve_windows([pinned] * 10, outputs=outs)
    e1.record(dp.stream); torch.cuda.synchronize()
    print(f"solve_windows x10: {e0.elapsed_time(e1)/10:.2f} ms/window device, {(time.perf_counter()-t0)*100:.2f} host")
# phases
import ctypes as C
from paper_2512_02293_b200 import _lib as L
for rep in range(2):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    L.check(dp.lib.vba_bind_inputs(dp.ctx, dp._sptr(), dp.d_tgt.data_ptr(), dp.d_w.data_ptr(), 1)); t.append(time.perf_counter())
    dp.load_state(); torch.cuda.synchronize(); t.append(time.perf_counter())
    dp.solve(); t.append(time.perf_counter())
    L.check(dp.lib.vba_download(dp.ctx, dp._sptr())); torch.cuda.synchronize(); t.append(time.perf_counter())
    print("bind %.2f load %.2f solve %.2f download %.2f ms" % tuple(1e3*(b-a) for a, b in zip(t, t[1:])))
