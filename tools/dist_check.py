"""Functional check of the edge-sharded multi-rank solve on whatever GPUs exist.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_check.py [cfg]

Ranks share GPUs round-robin; with fewer GPUs than ranks the collective runs over gloo
(host-mediated: no kernel ever waits on another rank's kernel), else NCCL.  Rank 0
compares the sharded solve (cost trajectory, states, all disparities) with a one-rank
solve: they must be bitwise equal."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02293_b200.device import DeviceProblem  # noqa: E402
from paper_2512_02293_b200.distributed import make_sharded_problem, partition_sources  # noqa: E402
from paper_2512_02293_b200.problem import pack_graph  # noqa: E402
from paper_2512_02293_b200.workloads import CONFIGS, make_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
ngpu = torch.cuda.device_count()
torch.cuda.set_device(rank % ngpu)
backend = "nccl" if world <= ngpu else "gloo"
dist.init_process_group(backend)
P = pack_graph(make_workload(cfg))
opts = {"max_iterations": CONFIGS[cfg].iterations}
dp = make_sharded_problem(P, opts, rank, world)
dp.load_state()
rep = dp.solve()
out = dp.download()
if rank == 0:
    ref = DeviceProblem(P, opts)
    ref.load_state()
    r1 = ref.solve()
    o1 = ref.download()
    dc = abs(rep["final_cost"] - r1["final_cost"]) / abs(r1["final_cost"])
    dpos = float(np.abs(out["p"] - o1["p"]).max())
    # every rank's disparities are gathered on download: compare all of them
    ddisp = float(np.abs(out["disp"] - o1["disp"]).max() / np.abs(o1["disp"]).max())
    same = (rep["cost_trajectory"] == r1["cost_trajectory"] and rep["iterations"] == r1["iterations"]
            and all(np.array_equal(out[k], o1[k]) for k in ("q", "p", "v", "bg", "ba", "disp", "grav_q")))
    print(f"world {world} ({backend}): cost {rep['final_cost']:.9e} vs {r1['final_cost']:.9e} (rel {dc:.2e}), "
          f"max |dp| {dpos:.2e}, disp rel {ddisp:.2e}, iterations {rep['iterations']}/{r1['iterations']}, "
          f"bitwise {same}, gathered {dp._collective.bytes / 1e6:.1f} MB in {dp._collective.calls} calls")
    # ranks gather each other's blocks and assemble in the single-GPU order: bitwise equal
    assert same, "sharded solve differs from the one-rank solve"
    assert dc == 0.0 and dpos == 0.0 and ddisp < 1e-5
    print("dist_check ok")
dist.barrier()
dist.destroy_process_group()
