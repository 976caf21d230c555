"""The CPU oracle (oracle/vi_ba.py) reproduces the reference's own outputs.

Golden vectors were produced by running the reference solver
(tests/golden/make_golden.py); this pins the restatement that the GPU parity
tests compare against.
"""
import copy

import numpy as np
import pytest

import oracle
from conftest import golden_names, load_golden

NAMES = golden_names()


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    s = max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / s)


@pytest.mark.parametrize("name", NAMES)
def test_energy_matches_reference(name):
    P, out, _ = load_golden(name)
    e = oracle.total_energy(P)
    assert abs(e - float(out["energy"])) <= 1e-10 * max(abs(float(out["energy"])), 1.0)


@pytest.mark.parametrize("name", NAMES)
def test_linearize_matches_reference(name):
    P, out, opts = load_golden(name)
    L = oracle.Layout(P, opts)
    H_pp, H_pd, H_dd, g_p, g_d = oracle.linearize_dense(P, L)
    assert rel(H_pp, out["H_pp"]) < 1e-12
    assert rel(H_pd, out["H_pd"]) < 1e-12
    assert rel(H_dd, out["H_dd"]) < 1e-12
    assert rel(g_p, out["g_p"]) < 1e-10
    assert rel(g_d, out["g_d"]) < 1e-10


@pytest.mark.parametrize("name", NAMES)
def test_solve_step_matches_reference(name):
    P, out, opts = load_golden(name)
    L = oracle.Layout(P, opts)
    lin = oracle.linearize_dense(P, L)
    dx, dxd = oracle.solve_step_dense(L, opts, *lin, opts["damping"])
    assert rel(dx, out["dx"]) < 1e-8
    assert rel(dxd, out["dxd"]) < 1e-8
    # sparse (per-keyframe) Schur restatement agrees with the dense one
    sp = oracle.linearize_sparse(P, L)
    dx2, dxd2 = oracle.solve_step_sparse(L, opts, *sp, opts["damping"])
    assert rel(dx2, out["dx"]) < 1e-8
    assert rel(dxd2, out["dxd"]) < 1e-8


@pytest.mark.parametrize("name", NAMES)
def test_solve_vi_ba_matches_reference(name):
    P, out, opts = load_golden(name)
    P = copy.deepcopy(P)
    rep = oracle.solve_vi_ba(P, opts)
    ref = out["report"]
    assert rep["iterations"] == ref["iterations"]
    assert rep["termination"] == ref["termination"]
    c0, c1 = np.array(rep["cost_trajectory"]), np.array(ref["cost_trajectory"])
    assert len(c0) == len(c1)
    assert np.all(np.abs(c0 - c1) <= 1e-6 * np.maximum(c1, 1e-3))
    for k in ("p", "v", "disp"):
        assert np.abs(P[k] - out["final_" + k]).max() < 1e-8, k


@pytest.mark.parametrize("cfg", [0, 1])
def test_sparse_oracle_matches_reference_at_baseline_config(cfg):
    """Pins the per-keyframe sparse restatement -- the oracle behind the config-4 golden, where
    the reference cannot run -- to the reference's own outputs at BASELINE shapes (full 48x64
    grids, out-degree 3 / 6): linearisation, Schur system, step (tests/golden/bcfg<cfg>.npz)."""
    from conftest import load_config_golden, packed_hash
    from oracle import vi_ba as V
    from paper_2512_02293_b200.problem import pack_graph
    from paper_2512_02293_b200.workloads import make_workload
    G = load_config_golden(cfg)
    P = pack_graph(make_workload(cfg))
    assert packed_hash(P) == G["meta"]["input_hash"]
    opts = dict(G["meta"]["opts"], frozen_keyframes=(0,))
    L = oracle.Layout(P, opts)
    H_pp, Hpd, H_dd, g_p, g_d = oracle.linearize_sparse(P, L)
    assert rel(H_pp, G["H_pp"]) < 1e-12 and rel(g_p, G["g_p"]) < 1e-10
    assert rel(H_dd, G["H_dd"]) < 1e-12 and rel(g_d, G["g_d"]) < 1e-10
    H, g, _ = V.reduced_system_sparse(L, opts, H_pp, Hpd, H_dd, g_p, g_d, opts["damping"])
    free = L.free_mask()
    assert rel(H[np.ix_(free, free)], G["Hred"]) < 1e-12 and rel(g[free], G["gred"]) < 1e-10
    dx, dxd = oracle.solve_step_sparse(L, opts, H_pp, Hpd, H_dd, g_p, g_d, opts["damping"])
    assert rel(dx, G["dx"]) < 1e-8 and rel(dxd, G["dxd"]) < 1e-8
