"""Drop-in replacement for ``vislam.solver.solve_vi_ba`` / ``total_energy``.

Same signatures and semantics as the reference
(/root/reference/pkg/src/vislam/solver.py:118-131, 344-411):

* ``solve_vi_ba(graph, opts=None) -> SolveReport`` minimises the joint vision
  + inertial energy in place: keyframe states, disparities and (with
  ``optimize_gravity``) the gravity direction are replaced by new objects of
  the graph's own classes; frozen keyframes keep their objects bit-identical.
  ``max_iterations=0`` echoes the initial cost and leaves the graph untouched.
* ``total_energy(graph) -> float``.

The graph may be built from the reference package's classes or from
``paper_2512_02293_b200.types``; it is read duck-typed.  All arithmetic runs
on the GPU through libvba (include/vba.h); this module packs (natively,
``csrc/vba_pack.cpp``, into page-locked buffers), uploads asynchronously, calls
``vba_solve`` (the native LM loop) and writes results back.

Contexts are cached by topology (keyframe pixel counts, edge list, IMU pairs,
frozen set, intrinsics, extrinsic, pixel grid, options): solving another window
of the same shape -- the tracker's steady state, or repeated solves of one
graph -- reuses the device workspace and the planner's schedules
(``DeviceProblem.rebind``) instead of rebuilding them.  ``clear_cache()`` frees them.
"""

from __future__ import annotations

import hashlib
from collections import OrderedDict

import numpy as np
import torch

from . import _lib as L
from .device import DeviceProblem, HostLayout
from .problem import options_dict, write_back
from .types import SolveOptions, SolveReport

__all__ = ["solve_vi_ba", "total_energy", "SolveOptions", "SolveReport", "clear_cache"]

_CACHE: "OrderedDict[tuple, DeviceProblem]" = OrderedDict()
CACHE_SIZE = 2


def clear_cache():
    while _CACHE:
        _, dp = _CACHE.popitem()
        dp.close()


def _topology_key(H: HostLayout, o: dict, dev: int):
    h = hashlib.blake2b(digest_size=16)
    for a in (H.npix, H.ei, H.ej, H.fi, H.fj, H.frozen, H.intr, H.Tcb):
        h.update(np.ascontiguousarray(a).tobytes())
        h.update(b"|")
    if H.pix is not None:                 # explicit coordinates: part of the static schedule's input
        h.update(np.ascontiguousarray(H.pix).tobytes())
    # the frozen set enters as the per-keyframe flags hashed above (kids change as a window slides)
    opts = tuple(sorted((k, tuple(v) if isinstance(v, (list, tuple)) else v) for k, v in o.items()
                        if k != "frozen_keyframes"))
    return (dev, H.K, H.E, H.F, H.mode, H.grid, H.has_Tcb, opts, h.hexdigest())


def _problem_for(graph, o: dict) -> DeviceProblem:
    if not L.cuda_available():
        raise RuntimeError("paper_2512_02293_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    H = HostLayout.from_graph(graph, o)
    dev = torch.cuda.current_device()
    key = _topology_key(H, o, dev)
    dp = _CACHE.pop(key, None)
    if dp is not None:
        dp.stream = torch.cuda.current_stream(dp.device)
        dp.rebind(H)
    else:
        dp = DeviceProblem(None, o, layout=H)
    _CACHE[key] = dp
    while len(_CACHE) > CACHE_SIZE:
        _CACHE.popitem(last=False)[1].close()
    return dp


def total_energy(graph) -> float:
    """solver.py:118-131 on the GPU (K2 vision energy + K3 inertial energy, fp64 sums)."""
    dp = _problem_for(graph, options_dict(SolveOptions(max_iterations=0)))
    return float(dp.energy()[0])


def solve_vi_ba(graph, opts=None) -> SolveReport:
    """solver.py:344-411 on the GPU; writes the solution back into ``graph`` in place."""
    if opts is None:
        opts = SolveOptions()
    o = options_dict(opts)
    dp = _problem_for(graph, o)
    rep = dp.solve()
    if rep["iterations"] > 0:
        s = dp.download()
        write_back(graph, s["q"], s["p"], s["v"], s["bg"], s["ba"], s["disp"], s["grav_q"], opts)
    return SolveReport(rep["iterations"], rep["initial_cost"], rep["final_cost"], rep["cost_trajectory"],
                       rep["termination"], rep["condition_warnings"])
