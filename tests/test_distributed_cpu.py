"""Edge-sharded decomposition of the reduced system, exercised with gloo (world_size 2) on CPU.

The CUDA path sums per-rank partial reduced systems with an all_reduce (NCCL on
the GPU box) and adds the ridge once (vba_host.cu, stage_step).  Here each rank
computes its partial with the oracle restricted to its edge/IMU shard, the
partials are all-reduced with gloo, and the result must equal the single-process
reduced system of solver.py:276-285.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import REPO, load_golden
from paper_2512_02293_b200.distributed import partition_sources, shard


def _sub_problem(P, edges, imus):
    Q = {k: v for k, v in P.items()}
    Q["ei"], Q["ej"] = P["ei"][edges], P["ej"][edges]
    segs = [(P["eoff"][e], P["eoff"][e + 1]) for e in edges]
    Q["eoff"] = np.concatenate([[0], np.cumsum([b - a for a, b in segs])]).astype(np.int64)
    for k in ("epix", "tgt", "w"):
        Q[k] = np.concatenate([P[k][a:b] for a, b in segs]) if segs else np.zeros((0, 2))
    for k in ("fi", "fj", "f_dt", "f_dR", "f_dp", "f_dv", "f_Jr", "f_Jp", "f_Jv", "f_cov", "f_bhat"):
        Q[k] = P[k][imus]
    return Q


def _partial(P, opts, rank, world, lam):
    edges, imus = shard(P, rank, world)
    Q = _sub_problem(P, edges, imus)
    L = oracle.Layout(Q, opts)
    lin = oracle.linearize_sparse(Q, L)
    H, g, _ = oracle.vi_ba.reduced_system_sparse(L, opts, *lin, lam)
    ridge = opts.get("ridge", 1e-10)
    H[np.diag_indices_from(H)] -= ridge            # ridge is added once, after the reduce
    e = oracle.total_energy(Q)
    return H, g, e


@pytest.mark.parametrize("name", ["win8_px30", "cfg0_grid12x16"])
@pytest.mark.parametrize("world", [2, 3])
def test_partition_covers_every_edge_once(name, world):
    P, _, _ = load_golden(name)
    parts = partition_sources(P, world)
    assert parts[0][0] == 0 and parts[-1][1] == len(P["kid"])
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    E = np.concatenate([shard(P, r, world)[0] for r in range(world)])
    F = np.concatenate([shard(P, r, world)[1] for r in range(world)])
    assert sorted(E.tolist()) == list(range(len(P["ei"])))
    assert sorted(F.tolist()) == list(range(len(P["fi"])))


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, _, opts = load_golden(name)
    lam = 1e-3
    H, g, e = _partial(P, opts, rank, world, lam)
    tH, tg, te = torch.from_numpy(H), torch.from_numpy(g), torch.tensor([e], dtype=torch.float64)
    for t in (tH, tg, te):
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    H = tH.numpy()
    H[np.diag_indices_from(H)] += opts.get("ridge", 1e-10)
    if rank == 0:
        q.put((H, tg.numpy(), float(te.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["win8_px30", "cfg0_grid12x16"])
def test_gloo_allreduce_of_partial_reduced_systems(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    H, g, e = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    P, _, opts = load_golden(name)
    L = oracle.Layout(P, opts)
    lin = oracle.linearize_sparse(P, L)
    Href, gref, _ = oracle.vi_ba.reduced_system_sparse(L, opts, *lin, 1e-3)
    assert np.abs(H - Href).max() <= 1e-9 * np.abs(Href).max()
    assert np.abs(g - gref).max() <= 1e-9 * np.abs(gref).max()
    eref = oracle.total_energy(P)
    assert abs(e - eref) <= 1e-12 * eref
