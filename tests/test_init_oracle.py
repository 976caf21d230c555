"""The stage-2 initialisation oracle (oracle/init.py) reproduces the reference's own
init_inertial_only (tests/golden/init, make_init_golden.py).

These windows are noise-free: both solvers drive the inertial energy to the fp64 floor
(1e-16 ... 1e-22 of the initial cost) and then stop on "no decrease at max damping", so the
iteration at which each one stops depends on summation order at that floor.  Costs are
compared while above 1e-9 of the initial one, the solution itself at fp64 tolerances."""
import numpy as np
import pytest

from conftest import init_golden_names, load_init_golden
from oracle import init as O

NAMES = [n for n in init_golden_names() if n != "full_pipeline"]


def costs_agree(c, cr, floor=1e-9, tol=1e-8):
    n = 0
    for a, b in zip(c, cr):
        if b < floor * cr[0]:
            break
        assert abs(a - b) <= tol * b, (a, b)
        n += 1
    return n


@pytest.mark.parametrize("name", NAMES)
def test_init_inertial_only_matches_reference(name):
    P, out = load_init_golden(name)
    s, grav, bias, vel, rep = O.init_inertial_only(P)
    ref = out["meta"]["reports"]["inertial"]
    assert costs_agree(rep["cost_trajectory"], ref["cost_trajectory"]) >= 2
    assert abs(s - float(out["log_scale"])) < 1e-9
    assert np.abs(bias - out["bias"]).max() < 1e-9
    assert np.abs(vel - out["velocities"]).max() < 1e-8
    assert np.abs(grav - out["grav_q"]).max() < 1e-10
