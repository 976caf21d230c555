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
