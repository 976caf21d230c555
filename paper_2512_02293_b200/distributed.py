"""Edge-sharded multi-GPU VI-BA (one process per GPU, NCCL over NVLink via torch.distributed).

Partition: every out-edge of source keyframe i lives on the
rank that owns i, so per-pixel disparity elimination, the Schur fill-in and the
back-substitution are rank-local.  Ranks own contiguous keyframe ranges balanced
by edge rows; IMU factor (i, i+1) belongs to the owner of i.  States are
replicated.

Exchange (include/vba.h, vba_problem.shard_* and vba_set_gather): every rank
holds the whole problem and plans the whole solve, but computes only its own
slices of the per-edge vision blocks, per-factor IMU blocks, per-source fill-in
blocks and per-tile energy partials.  The native LM loop all-gathers those slices
(once per linearisation for the vision/IMU blocks, once per trial for the fill-in
and energies) and every rank then assembles, in the single-GPU order, the
identical reduced system and runs the identical Cholesky: an N-rank solve is
bitwise the 1-rank solve (deterministic, rank-count invariant), and it moves the
compact blocks (≈ 50 MB per trial at config 4) instead of all-reducing the dense
reduced system (235 MB).  The step norm is max-reduced; the disparities each rank
updated are gathered on download.

The hooks run their collectives on the solve's own CUDA stream
(``torch.cuda.ExternalStream``), so they are ordered after the kernels that wrote
the slices whatever torch's current stream is.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def partition_sources(P, world: int):
    """Contiguous keyframe ranges [k0, k1) per rank, balanced by edge rows."""
    K = len(P["kid"])
    ei = np.asarray(P["ei"], np.int64)
    rows = np.diff(np.asarray(P["eoff"], np.int64))
    work = np.bincount(ei, weights=rows, minlength=K).astype(float) + 1.0
    cum = np.concatenate([[0.0], np.cumsum(work)])
    tot = cum[-1]
    bounds = [0]
    for r in range(1, world):
        bounds.append(int(np.searchsorted(cum, tot * r / world, side="left")))
    bounds.append(K)
    bounds = np.maximum.accumulate(np.clip(bounds, 0, K))
    return [(int(bounds[r]), int(bounds[r + 1])) for r in range(world)]


def shard_bounds(P, world: int):
    """Keyframe bounds kb[world + 1] of partition_sources (vba_problem.h_shard_kbounds)."""
    parts = partition_sources(P, world)
    return np.array([p[0] for p in parts] + [parts[-1][1]], dtype=np.int32)


def shard(P, rank: int, world: int):
    """(edge indices, IMU factor indices) owned by ``rank``."""
    k0, k1 = partition_sources(P, world)[rank]
    ei = np.asarray(P["ei"], np.int64)
    fi = np.asarray(P["fi"], np.int64)
    edges = np.nonzero((ei >= k0) & (ei < k1))[0]
    imu = np.nonzero((fi >= k0) & (fi < k1))[0]
    return edges, imu


class _CudaView:
    """Zero-copy view of a device buffer for torch (``__cuda_array_interface__``)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


class TorchCollective:
    """vba_allreduce_fn / vba_allgather_fn backed by torch.distributed.

    NCCL: collectives on the solve stream; variable-size gathers through one padded
    all_gather_into_tensor.  gloo (ranks sharing a GPU in tools/dist_check.py, or CPU
    process groups): host-staged, so no kernel ever waits on another rank's kernel."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.device = device
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.calls = 0
        self.bytes = 0

        def _reduce(user, buf, count, op, stream):
            try:
                with self._on(stream):
                    t = self.torch.as_tensor(_CudaView(buf, count), device=self.device)
                    red = self.dist.ReduceOp.SUM if op == 0 else self.dist.ReduceOp.MAX
                    if self.nccl:
                        self.dist.all_reduce(t, op=red, group=self.group)
                    else:
                        h = t.cpu()
                        self.dist.all_reduce(h, op=red, group=self.group)
                        t.copy_(h)
                self.calls += 1
                self.bytes += 8 * int(count)
                return 0
            except Exception as exc:  # never raise through the C ABI
                print(f"[vba] allreduce failed: {exc}")
                return 1

        def _gather(user, buf, offs, world, stream):
            try:
                o = [int(offs[r]) for r in range(world + 1)]
                self._gather(buf, o, world, stream)
                self.calls += 1
                return 0
            except Exception as exc:
                print(f"[vba] gather failed: {exc}")
                return 1

        self._cfn = L.ALLREDUCE_FN(_reduce)
        self._gfn = L.ALLGATHER_FN(_gather)

    def _on(self, stream):
        torch = self.torch
        if stream:
            return torch.cuda.stream(torch.cuda.ExternalStream(int(stream), device=self.device))
        import contextlib
        return contextlib.nullcontext()

    def _gather(self, buf, o, world, stream):
        torch, dist = self.torch, self.dist
        sizes = [o[r + 1] - o[r] for r in range(world)]
        m = max(sizes)
        if m == 0:
            return
        base = o[0]
        with self._on(stream):
            full = torch.as_tensor(_CudaView(buf + 8 * base, o[-1] - base), device=self.device)
            mine = full[o[self.rank] - base:o[self.rank + 1] - base]
            if self.nccl:
                if all(s == m for s in sizes):
                    dist.all_gather_into_tensor(full, mine.clone(), group=self.group)
                else:
                    tmp = torch.empty(world * m, dtype=full.dtype, device=full.device)
                    tmp[self.rank * m:self.rank * m + sizes[self.rank]].copy_(mine)
                    dist.all_gather_into_tensor(tmp, tmp[self.rank * m:(self.rank + 1) * m].clone(),
                                                group=self.group)
                    for r in range(world):
                        if r != self.rank and sizes[r]:
                            full[o[r] - base:o[r + 1] - base].copy_(tmp[r * m:r * m + sizes[r]])
            else:
                h = torch.zeros(m, dtype=torch.float64)
                h[:sizes[self.rank]].copy_(mine)
                parts = [torch.empty(m, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, h, group=self.group)
                for r in range(world):
                    if r != self.rank and sizes[r]:
                        full[o[r] - base:o[r + 1] - base].copy_(parts[r][:sizes[r]])
        self.bytes += 8 * int(o[-1] - base)

    def attach(self, dp):
        L.check(dp.lib.vba_set_collective(dp.ctx, self._cfn, None))
        L.check(dp.lib.vba_set_gather(dp.ctx, self._gfn, None))


def make_sharded_problem(P, opts, rank, world, group=None):
    """DeviceProblem of the whole problem owning the source keyframes of ``rank``, with the
    torch.distributed hooks attached (a plain single-GPU problem when world == 1)."""
    from .device import DeviceProblem, HostLayout
    H = HostLayout(P, opts)
    if world <= 1:
        return DeviceProblem(P, opts, layout=H)
    dp = DeviceProblem(P, opts, layout=H, shard=(rank, world, shard_bounds(P, world)))
    coll = TorchCollective(group=group, device=dp.device)
    coll.attach(dp)
    dp._collective = coll
    return dp
