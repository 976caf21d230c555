"""Time the device PGBA solve on make_pgba_workload() (for launch-list profiling)."""
import copy
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02293_b200.pgba import DevicePoseGraph, pack_pose_graph  # noqa: E402
from paper_2512_02293_b200.workloads import make_pgba_workload  # noqa: E402

g, _ = make_pgba_workload()
P = pack_pose_graph(g)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    dp = DevicePoseGraph(copy.deepcopy(P), {"max_iterations": 6})
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = dp.solve()
    e1.record()
    torch.cuda.synchronize()
    print(f"pgba solve {e0.elapsed_time(e1):.2f} ms, {r['iterations']} it, trials {r.get('trials')}, {r['termination']}")
    dp.close()
