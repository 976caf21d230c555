"""The drop-in entry point on the GPU: ``paper_2512_02293_b200.solver.solve_vi_ba(graph, opts)``.

Two kinds of checks, both through the public call a vislam user makes (graph in,
SolveReport out, graph written back in place):

* the reference's own solver contract, /root/reference/pkg/tests/test_solver.py
  :17-175, on the same windows (its fixtures and seeds, run through the
  reference by tests/golden/make_contract_golden.py): zero-iteration echo,
  recovery, strictly decreasing trajectory, IMU-only convergence, Schur == dense,
  bit-identical gauge keyframe, determinism, gravity optimisation;
* the SolveReport and final states against the reference's, on the BASELINE
  windows (configs 0 and 1, goldens by the reference) and the small goldens.

Those contract windows are noise-free: the reference drives their energy to the
fp64 floor (1e-8 ... 1e-21).  The GPU evaluates per-pixel residuals in fp32
(north_star), which resolves a residual to ~1e-7 of the flow, so near the optimum
its energies and steps follow the reference only down to an absolute floor:
costs are compared entrywise to 1e-6 relative plus ``FP32_FLOOR`` x the initial
cost (measured worst case on these windows: 2e-10 x), and iteration counts /
terminations are compared only on the noisy BASELINE windows, where the costs stay
far above that floor.  The contract properties themselves are asserted as the
reference states them.
"""
import copy

import numpy as np
import pytest

from conftest import config_golden_names, graph_from_packed, load_config_golden, load_contract, packed_hash

pytestmark = pytest.mark.gpu

FP32_FLOOR = 1e-9
TOL_COST = 1e-6


def _solver():
    from paper_2512_02293_b200 import solver
    return solver


def _opts(meta, **kw):
    from paper_2512_02293_b200.types import SolveOptions
    o = dict(meta["opts"])
    o.update(kw)
    return SolveOptions(**o)


def _costs_agree(rep, ref):
    """Accepted costs agree entrywise to 1e-6 relative plus an absolute fp32 floor of
    FP32_FLOOR x the initial cost; returns how many entries were compared."""
    c, cr = list(rep.cost_trajectory), list(ref["cost_trajectory"])
    print(f"  ours {['%.6e' % v for v in c]} {rep.iterations} it {rep.termination}\n"
          f"  ref  {['%.6e' % v for v in cr]} {ref['iterations']} it {ref['termination']}")
    floor = FP32_FLOOR * cr[0]
    n = 0
    for a, b in zip(c, cr):
        assert abs(a - b) <= TOL_COST * b + floor, (a, b)
        n += 1
    return n


def test_zero_iterations_echoes_initial_cost(cuda_ok):
    """test_solver.py:58-68"""
    S = _solver()
    P, out, meta = load_contract("zero_iterations")
    g = graph_from_packed(P)
    before = [kf.state.pose.translation.copy() for kf in g.keyframes]
    c0 = S.total_energy(g)
    rep = S.solve_vi_ba(g, _opts(meta))
    assert rep.iterations == 0 and rep.termination == "max_iterations"
    assert rep.initial_cost == rep.final_cost == c0
    assert rep.cost_trajectory == [c0]
    for kf, p in zip(g.keyframes, before):
        assert np.all(kf.state.pose.translation == p)
    assert abs(c0 - float(out["energy"])) <= TOL_COST * float(out["energy"])


def test_recovers_perturbed_window(cuda_ok):
    """test_solver.py:71-77: ATE <= 1e-5 m within 15 iterations."""
    S = _solver()
    P, out, meta = load_contract("recovers_perturbed")
    g = graph_from_packed(P)
    rep = S.solve_vi_ba(g, _opts(meta))
    ate = float(np.sqrt(np.mean(np.sum((np.array([kf.state.pose.translation for kf in g.keyframes])
                                        - out["truth_p"]) ** 2, axis=1))))
    print(f"recovers: ATE {ate:.2e} m")
    _costs_agree(rep, meta["report"])
    assert rep.iterations <= 15
    assert ate <= 1e-5


def test_cost_trajectory_strictly_decreasing(cuda_ok):
    """test_solver.py:80-87"""
    S = _solver()
    P, out, meta = load_contract("strictly_decreasing")
    g = graph_from_packed(P)
    rep = S.solve_vi_ba(g, _opts(meta))
    c = rep.cost_trajectory
    assert all(c[k + 1] < c[k] for k in range(len(c) - 1))
    assert abs(rep.final_cost - S.total_energy(g)) <= 1e-10 * max(rep.final_cost, 1.0)
    assert _costs_agree(rep, meta["report"]) >= 3


def test_zero_weight_vision_drives_inertial_to_zero(cuda_ok):
    """test_solver.py:90-103 (vision weights 0: the total energy is the inertial energy)."""
    S = _solver()
    P, out, meta = load_contract("zero_weight_vision")
    g = graph_from_packed(P)
    rep = S.solve_vi_ba(g, _opts(meta))
    e = S.total_energy(g)
    print(f"zero-weight vision: inertial energy {e:.3e}")
    _costs_agree(rep, meta["report"])
    assert e <= 1e-10


@pytest.mark.parametrize("name", ["schur_dense_3_20", "schur_dense_5_50", "schur_dense_4_7"])
def test_schur_step_matches_dense_step(name, cuda_ok):
    """test_solver.py:106-121: 3 iterations with use_schur True / False agree to 1e-8.

    Poses and velocities are held to the reference's 1e-8 (measured <= 1e-8, 1e-10 typical).
    Disparities are held to 1e-6 of their magnitude: the per-pixel g_d / H_dd come from fp32
    residuals, which on these noise-free 640x480 / fx = 300 windows resolve r to ~1e-6 px near
    the optimum, i.e. ~1e-7 in d after each step -- for either path, and against the
    reference's own Schur and dense solves alike (both printed)."""
    from paper_2512_02293_b200.types import Rotation
    S = _solver()
    P, out, meta = load_contract(name)
    gs = graph_from_packed(P)
    gd = graph_from_packed(P)
    S.solve_vi_ba(gs, _opts(meta, use_schur=True))
    S.solve_vi_ba(gd, _opts(meta, use_schur=False))
    worst = 0.0
    for a, b in zip(gs.keyframes, gd.keyframes):
        worst = max(worst, np.abs(a.state.pose.translation - b.state.pose.translation).max(),
                    Rotation(a.state.pose.rotation.q).angle_to(Rotation(b.state.pose.rotation.q)),
                    np.abs(a.state.velocity - b.state.velocity).max())
    # and both against the reference's Schur and dense solves
    pr = np.abs(np.array([kf.state.pose.translation for kf in gs.keyframes]) - out["final_p"]).max()
    pd = np.abs(np.array([kf.state.pose.translation for kf in gd.keyframes]) - out["dense_p"]).max()
    ds = np.abs(np.concatenate([kf.disparities for kf in gs.keyframes]) - out["final_disp"]).max()
    dd = np.abs(np.concatenate([kf.disparities for kf in gd.keyframes]) - out["dense_disp"]).max()
    dv = max(np.abs(a.state.velocity - b.state.velocity).max() for a, b in zip(gs.keyframes, gd.keyframes))
    ddp = max(np.abs(a.disparities - b.disparities).max() for a, b in zip(gs.keyframes, gd.keyframes))
    print(f"{name}: schur-vs-dense poses {worst:.2e} (velocity {dv:.2e}, disparity {ddp:.2e}); vs reference: "
          f"translation schur {pr:.2e} dense {pd:.2e}, disparity schur {ds:.2e} dense {dd:.2e}")
    dmax = np.abs(out["final_disp"]).max()
    assert worst <= 1e-8
    assert ddp <= 1e-6 * dmax and ds <= 1e-6 * dmax and dd <= 1e-6 * dmax


def test_frozen_blocks_bit_identical(cuda_ok):
    """test_solver.py:124-138"""
    S = _solver()
    P, out, meta = load_contract("frozen_bit_identical")
    g = graph_from_packed(P)
    fr = g.keyframes[0].state
    b = (fr.pose.rotation.q.tobytes(), fr.pose.translation.tobytes(), fr.velocity.tobytes(),
         fr.bias.vector().tobytes())
    rep = S.solve_vi_ba(g, _opts(meta))
    af = g.keyframes[0].state
    assert rep.iterations > 0
    assert (af.pose.rotation.q.tobytes(), af.pose.translation.tobytes(), af.velocity.tobytes(),
            af.bias.vector().tobytes()) == b


def test_solver_is_deterministic(cuda_ok):
    """test_solver.py:141-153 (the second solve reuses the cached context: rebind path)."""
    S = _solver()
    P, out, meta = load_contract("deterministic")
    g1 = graph_from_packed(P)
    g2 = graph_from_packed(P)
    r1 = S.solve_vi_ba(g1, _opts(meta))
    r2 = S.solve_vi_ba(g2, _opts(meta))
    assert r1.cost_trajectory == r2.cost_trajectory
    for a, b in zip(g1.keyframes, g2.keyframes):
        assert a.state.pose.rotation.q.tobytes() == b.state.pose.rotation.q.tobytes()
        assert a.state.pose.translation.tobytes() == b.state.pose.translation.tobytes()
        assert a.disparities.tobytes() == b.disparities.tobytes()


def test_gravity_gauge_optimization_reduces_energy(cuda_ok):
    """test_solver.py:165-175"""
    S = _solver()
    P, out, meta = load_contract("gravity_optimization")
    g = graph_from_packed(P)
    e0 = S.total_energy(g)
    rep = S.solve_vi_ba(g, _opts(meta))
    e1 = S.total_energy(g)
    print(f"gravity: {e0:.3e} -> {e1:.3e}")
    _costs_agree(rep, meta["report"])
    assert e1 < e0 * 1e-3


def test_write_back_objects(cuda_ok):
    """New objects of the graph's own classes for free keyframes (solver.py:326-341); the
    gauge keyframe keeps its object; disparities replaced for every keyframe."""
    S = _solver()
    P, out, meta = load_contract("frozen_bit_identical")
    g = graph_from_packed(P)
    old = [kf.state for kf in g.keyframes]
    oldd = [kf.disparities for kf in g.keyframes]
    S.solve_vi_ba(g, _opts(meta))
    assert g.keyframes[0].state is old[0]
    for kf, s, d in zip(g.keyframes[1:], old[1:], oldd[1:]):
        assert kf.state is not s and type(kf.state) is type(s)
        assert type(kf.state.pose) is type(s.pose) and kf.disparities is not d


@pytest.mark.parametrize("cfg", [c for c in config_golden_names() if c <= 1])
def test_dropin_matches_reference_at_baseline_config(cfg, cuda_ok):
    """graph -> SolveReport through the drop-in on BASELINE configs 0 and 1 (reference goldens):
    identical iterations, termination and warnings; every cost within 1e-6; final states."""
    from paper_2512_02293_b200.problem import pack_graph
    from paper_2512_02293_b200.types import SolveOptions
    from paper_2512_02293_b200.workloads import make_workload
    S = _solver()
    G = load_config_golden(cfg)
    g = make_workload(cfg)
    assert packed_hash(pack_graph(g)) == G["meta"]["input_hash"]
    o = dict(G["meta"]["opts"])
    o["frozen_keyframes"] = tuple(o["frozen_keyframes"])
    rep = S.solve_vi_ba(g, SolveOptions(**o))
    ref = G["meta"]["report"]
    assert rep.iterations == ref["iterations"] and rep.termination == ref["termination"]
    assert rep.condition_warnings == ref["condition_warnings"]
    assert _costs_agree(rep, ref) == len(ref["cost_trajectory"]) == len(rep.cost_trajectory)
    F = pack_graph(g)
    for k in ("p", "v"):
        moved = np.abs(G["final_" + k] - pack_graph(make_workload(cfg))[k]).max()
        assert np.abs(F[k] - G["final_" + k]).max() <= 1e-5 * moved
    d = F["disp"]
    assert np.abs(d - G["final_disp"]).max() <= 1e-5 * G["final_disp_maxabs"]
