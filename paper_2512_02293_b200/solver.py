"""Drop-in replacement for ``vislam.solver.solve_vi_ba`` / ``total_energy``.

Same signatures and semantics as the reference
(/root/reference/pkg/src/vislam/solver.py:118-131, 344-411):

* ``solve_vi_ba(graph, opts=None) -> SolveReport`` minimises the joint vision
  + inertial energy in place: keyframe states, disparities and (with
  ``optimize_gravity``) the gravity direction are replaced by new objects of
  the graph's own classes; frozen keyframes keep their objects bit-identical.
* ``total_energy(graph) -> float``.

The graph may be built from the reference package's classes or from
``paper_2512_02293_b200.types``; it is read duck-typed.  All arithmetic runs
on the GPU through libvba (include/vba.h); this module only packs, uploads,
calls ``vba_solve`` (the native LM loop) and writes results back.
"""

from __future__ import annotations

from .device import DeviceProblem
from .problem import options_dict, pack_graph, write_back
from .types import SolveOptions, SolveReport

__all__ = ["solve_vi_ba", "total_energy", "SolveOptions", "SolveReport"]


def total_energy(graph) -> float:
    P = pack_graph(graph)
    dp = DeviceProblem(P, {"max_iterations": 0})
    try:
        return float(dp.energy()[0])
    finally:
        dp.close()


def solve_vi_ba(graph, opts=None) -> SolveReport:
    if opts is None:
        opts = SolveOptions()
    o = options_dict(opts)
    P = pack_graph(graph)
    dp = DeviceProblem(P, o)
    try:
        rep = dp.solve()
        if rep["iterations"] > 0:
            s = dp.download()
            write_back(graph, s["q"], s["p"], s["v"], s["bg"], s["ba"], s["disp"], s["grav_q"], opts)
    finally:
        dp.close()
    return SolveReport(rep["iterations"], rep["initial_cost"], rep["final_cost"], rep["cost_trajectory"],
                       rep["termination"], rep["condition_warnings"])
