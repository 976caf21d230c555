"""Edge-sharded multi-GPU VI-BA (one process per GPU, NCCL over NVLink via torch.distributed).

Partition: every out-edge of source keyframe i lives on the
rank that owns i, so per-pixel disparity elimination, the Schur fill-in and the
back-substitution are rank-local.  Ranks own contiguous keyframe ranges balanced
by edge rows; IMU factor (i, i+1) belongs to the owner of i.  States are
replicated.  Per LM trial the native driver calls the collective hook for

  * all_reduce(SUM) of the partial reduced system H_red, g_red (fp64), then the
    ridge is added once and every rank runs the identical Cholesky;
  * all_reduce(SUM) of the energy partials and all_reduce(MAX) of the step norm,

so every rank takes the same accept/reject decision (solver.py:383-398).
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
    """vba_allreduce_fn backed by torch.distributed (NCCL on GPUs, gloo on CPU tests)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.device = device
        self.calls = 0
        self.bytes = 0

        def _fn(user, buf, count, op, stream):
            try:
                t = self.torch.as_tensor(_CudaView(buf, count), device=self.device)
                red = self.dist.ReduceOp.SUM if op == 0 else self.dist.ReduceOp.MAX
                self.dist.all_reduce(t, op=red, group=self.group)
                self.calls += 1
                self.bytes += 8 * int(count)
                return 0
            except Exception as exc:  # never raise through the C ABI
                print(f"[vba] allreduce failed: {exc}")
                return 1

        self._cfn = L.ALLREDUCE_FN(_fn)

    def attach(self, dp):
        L.check(dp.lib.vba_set_collective(dp.ctx, self._cfn, None))


def make_sharded_problem(P, opts, rank, world, group=None):
    """DeviceProblem holding this rank's edge shard, with the NCCL hook attached."""
    from .device import DeviceProblem, HostLayout
    edges, imu = shard(P, rank, world)
    H = HostLayout(P, opts, edge_subset=edges, imu_subset=imu)
    dp = DeviceProblem(P, opts, layout=H)
    if world > 1:
        coll = TorchCollective(group=group, device=dp.device)
        coll.attach(dp)
        dp._collective = coll
    return dp
