"""The PGBA oracle (oracle/pgba.py) reproduces the reference's own outputs
(tests/golden/pgba, produced by vislam.loopclosure in make_pgba_golden.py)."""
import copy

import numpy as np
import pytest

from conftest import load_pgba_golden, pgba_golden_names
from oracle import pgba as O
from oracle import vi_ba as V

NAMES = pgba_golden_names()


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    s = max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / s)


@pytest.mark.parametrize("name", NAMES)
def test_energy_linearize_step(name):
    P, out, meta = load_pgba_golden(name)
    e = O.pg_energy(P)
    assert abs(e - float(out["energy"])) <= 1e-10 * max(float(out["energy"]), 1.0)
    L = O.PgLayout(P)
    H_pp, H_pd, H_dd, g_p, g_d = O.linearize_pg(P, L)
    assert rel(H_pp, out["H_pp"]) < 1e-12 and rel(g_p, out["g_p"]) < 1e-10
    if "H_pd" in out:
        assert rel(H_pd[:, out["H_pd_cols"]], out["H_pd"]) < 1e-12
        assert rel(H_dd, out["H_dd"]) < 1e-12 and rel(g_d, out["g_d"]) < 1e-10
    dx, dxd = V.solve_step_dense(L, meta["opts"], H_pp, H_pd, H_dd, g_p, g_d, meta["opts"]["damping"], True)
    assert rel(dx, out["dx"]) < 1e-8
    if len(dxd):
        assert rel(dxd, out["dxd"]) < 1e-8


@pytest.mark.parametrize("name", [n for n in NAMES if n != "stress"])
def test_solve_pgba(name):
    P, out, meta = load_pgba_golden(name)
    Q = copy.deepcopy(P)
    rep = O.solve_pgba(Q, meta["opts"])
    ref = meta["report"]
    assert rep["iterations"] == ref["iterations"] and rep["termination"] == ref["termination"]
    c, cr = np.array(rep["cost_trajectory"]), np.array(ref["cost_trajectory"])
    assert len(c) == len(cr) and np.all(np.abs(c - cr) <= 1e-8 * np.maximum(cr, 1e-6))
    assert np.abs(Q["st"] - out["final_st"]).max() < 1e-9
    assert np.abs(Q["ss"] - out["final_ss"]).max() < 1e-9
