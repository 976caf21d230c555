"""Edge-sharded decomposition of the reduced system, exercised with gloo (world_size 2-3) on CPU.

The CUDA path (vba_host.cu, paper_2512_02293_b200.distributed) has every rank compute
only the blocks it owns -- per-edge vision blocks of its source keyframes' out-edges,
per-factor IMU blocks of its factors, per-source Schur fill-in of its sources -- then
all-gathers them, and every rank assembles the reduced system in the single-GPU order.
Here each rank computes its owned blocks with the oracle, the blocks are all-gathered
with gloo, and the assembled system must be BITWISE the single-process assembly of
solver.py:276-285 (ownership covers every block exactly once, order preserved).
"""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import load_golden
from paper_2512_02293_b200.distributed import partition_sources, shard, shard_bounds


def _owned_blocks(P, opts, lam, k0, k1):
    """Blocks owned by the keyframe range [k0, k1): {("e", e): (i, j, Hii, Hjj, Hij, gi, gj)},
    {("f", f): IMU blocks}, {("s", n): (keyframes, fill block, fill gradient)}."""
    L = oracle.Layout(P, opts)
    ridge = opts.get("ridge", 1e-10)
    out = {}
    ei = np.asarray(P["ei"])
    coup = {}
    for e in np.nonzero((ei >= k0) & (ei < k1))[0]:
        i, j = int(P["ei"][e]), int(P["ej"][e])
        r, Ji, Jj, Jd, _ = oracle.vision_residual(P, e)
        out[("e", int(e))] = (i, j, np.einsum("nka,nkb->ab", Ji, Ji), np.einsum("nka,nkb->ab", Jj, Jj),
                              np.einsum("nka,nkb->ab", Ji, Jj), np.einsum("nka,nk->a", Ji, r),
                              np.einsum("nka,nk->a", Jj, r))
        c = coup.setdefault(i, {"Hdd": 0.0, "gd": 0.0, "B": {}})
        c["Hdd"] = c["Hdd"] + np.einsum("nk,nk->n", Jd, Jd)
        c["gd"] = c["gd"] + np.einsum("nk,nk->n", Jd, r)
        for kf, J in ((i, Ji), (j, Jj)):
            blk = np.einsum("nka,nk->an", J, Jd)
            c["B"][kf] = c["B"][kf] + blk if kf in c["B"] else blk
    for f in np.nonzero((np.asarray(P["fi"]) >= k0) & (np.asarray(P["fi"]) < k1))[0]:
        out[("f", int(f))] = (int(P["fi"][f]), int(P["fj"][f])) + tuple(oracle.vi_ba._imu_blocks(P, L, f))
    for n in sorted(coup):
        c = coup[n]
        inv = 1.0 / (c["Hdd"] * (1.0 + lam) + ridge)
        kfs = sorted(c["B"])
        B = np.concatenate([c["B"][k] for k in kfs], axis=0)
        out[("s", n)] = (kfs, (B * inv) @ B.T, B @ (inv * c["gd"]))
    return out


def _assemble(P, opts, lam, blocks):
    """Reduced system (before freezing) from the blocks, in the single-GPU order: edges by
    index, then IMU factors, then fill-in per source keyframe."""
    L = oracle.Layout(P, opts)
    npv, sd = L.npv, L.sdof
    H = np.zeros((npv, npv))
    g = np.zeros(npv)
    for key in sorted(k for k in blocks if k[0] == "e"):
        i, j, Hii, Hjj, Hij, gi, gj = blocks[key]
        ci, cj = L.cols(i, 0, 6), L.cols(j, 0, 6)
        H[np.ix_(ci, ci)] += Hii
        H[np.ix_(cj, cj)] += Hjj
        H[np.ix_(ci, cj)] += Hij
        H[np.ix_(cj, ci)] += Hij.T
        g[ci] += gi
        g[cj] += gj
    for key in sorted(k for k in blocks if k[0] == "f"):
        i, j, r, Ji, Jj, Jg = blocks[key]
        ci, cj = L.cols(i, 0, sd), L.cols(j, 0, sd)
        H[np.ix_(ci, ci)] += Ji.T @ Ji
        H[np.ix_(cj, cj)] += Jj.T @ Jj
        H[np.ix_(ci, cj)] += Ji.T @ Jj
        H[np.ix_(cj, ci)] += (Ji.T @ Jj).T
        g[ci] += Ji.T @ r
        g[cj] += Jj.T @ r
    idx = np.arange(npv)
    H[idx, idx] = H[idx, idx] * (1.0 + lam) + opts.get("ridge", 1e-10)
    for key in sorted(k for k in blocks if k[0] == "s"):
        kfs, F, gr = blocks[key]
        cols = np.concatenate([L.cols(k, 0, 6) for k in kfs])
        H[np.ix_(cols, cols)] -= F
        g[cols] -= gr
    return H, g


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
    kb = shard_bounds(P, world)
    mine = _owned_blocks(P, opts, 1e-3, int(kb[rank]), int(kb[rank + 1]))
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    blocks = {}
    for p in parts:
        assert not (set(p) & set(blocks)), "a block is owned by two ranks"
        blocks.update(p)
    H, g = _assemble(P, opts, 1e-3, blocks)
    if rank == 0:
        q.put((H, g))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("win8_px30", 2), ("cfg0_grid12x16", 2), ("cfg0_grid12x16", 3)])
def test_gloo_gathered_blocks_assemble_the_single_process_system_bitwise(name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world + (os.getpid() % 2000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    H, g = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    P, _, opts = load_golden(name)
    K = len(P["kid"])
    Hs, gs = _assemble(P, opts, 1e-3, _owned_blocks(P, opts, 1e-3, 0, K))
    assert np.array_equal(H, Hs) and np.array_equal(g, gs)
    # and the assembly is the reference's Schur system (oracle restatement, solver.py:276-285)
    L = oracle.Layout(P, opts)
    lin = oracle.linearize_sparse(P, L)
    Href, gref, _ = oracle.vi_ba.reduced_system_sparse(L, opts, *lin, 1e-3)
    assert np.abs(H - Href).max() <= 1e-9 * np.abs(Href).max()
    assert np.abs(g - gref).max() <= 1e-9 * np.abs(gref).max()
