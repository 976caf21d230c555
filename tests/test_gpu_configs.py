"""GPU parity at the BASELINE configs, through the kernel paths the bench times.

Goldens (tests/golden/bcfg<cfg>.npz, tests/golden/make_config_golden.py): the
reference itself at configs 0-3 (vislam, imported read-only in the build
container), the pinned sparse restatement oracle/vi_ba.py at config 4 (where the
reference's dense H_pd would need 96.6 GB).  The inputs are regenerated here with
the seeded workload generator and identified by their sha256 first.

What these windows exercise that the small fixtures do not: full 1024-pixel K1
tiles with the 4x16 blocked pixel mapping and split-tile adds (3072 and 12288
pixels per keyframe), per-edge fp32 partials of 256 pixels, Schur Gram tiles at
out-degree 6-30 (config 3/4 loop edges), and the 15- and 60-tile tensor-core
Cholesky of the reduced system (configs 3 and 4).

Tolerances are the north_star's, graded per block family with
no conditioning-based relaxation:

* H and g (vision family = H - H_imu, and the totals; H_dd, g_d, coupling H_pd;
  the reduced system H_red, g_red): max|Δ| / max|ref| <= 1e-4
* pose and disparity updates dx, dx_d: <= 1e-5
* full LM solves: identical iterations and termination, every accepted cost
  within 1e-6 relative, final states within the update tolerance.
"""
import copy

import numpy as np
import pytest

import oracle
from conftest import config_golden_names, golden_proj_vector, load_config_golden, packed_hash

pytestmark = pytest.mark.gpu

CFGS = config_golden_names()
TOL_H = 1e-4
TOL_DX = 1e-5
TOL_COST = 1e-6

_problems = {}


def problem(cfg):
    """(packed inputs, golden) for config ``cfg``; the inputs must hash to the golden's."""
    if cfg not in _problems:
        from paper_2512_02293_b200.problem import pack_graph
        from paper_2512_02293_b200.workloads import make_workload
        G = load_config_golden(cfg)
        P = pack_graph(make_workload(cfg))
        assert packed_hash(P) == G["meta"]["input_hash"], "workload generator drifted from the golden's inputs"
        _problems[cfg] = (P, G)
    return _problems[cfg]


def opts_of(G):
    o = dict(G["meta"]["opts"])
    o["frozen_keyframes"] = tuple(o["frozen_keyframes"])
    return o


def vec_err(G, name, ours):
    """max|Δ| / max|ref| over the stored (full or sampled) entries of a per-pixel vector."""
    ours = np.asarray(ours, float)
    assert len(ours) == int(G[name + "_n"])
    sel = ours[G[name + "_idx"]] if (name + "_idx") in G else ours
    return float(np.abs(sel - G[name]).max() / G[name + "_maxabs"])


def mat_err(G, name, ours, sdof=15):
    """Relative error of a pose-space matrix (whole, or over the stored blocks) and of its
    seeded-projection checksum |Δ(M v)| / (max|M| ||v||_1) (implied by the entrywise bound)."""
    ours = np.asarray(ours, float)
    n = int(G[name + "_n"])
    assert ours.shape == (n, n)
    scale = float(G[name + "_maxabs"])
    seed = {"H_pp": 11, "Hred": 12}[name]
    v = golden_proj_vector(n, seed)
    proj = float(np.abs(ours @ v - G[name + "_proj"]).max() / (scale * np.abs(v).sum()))
    if name in G:
        return float(np.abs(ours - G[name]).max() / scale), proj
    Kb = n // sdof
    B = ours.reshape(Kb, sdof, Kb, sdof)
    err = 0.0
    diag = np.stack([B[k, :, k, :] for k in range(Kb)])
    sub_ = np.stack([B[k + 1, :, k, :] for k in range(Kb - 1)])
    err = max(err, np.abs(diag - G[name + "_diag"]).max(), np.abs(sub_ - G[name + "_sub"]).max())
    for (a, b), blk in zip(G[name + "_oidx"], G[name + "_oblk"]):
        err = max(err, np.abs(B[a, :6, b, :6] - blk).max())
        assert np.all(B[a, :, b, :][6:, :] == 0) and np.all(B[a, :, b, :][:, 6:] == 0)
    return float(err / scale), proj


def _dp(P, opts):
    from paper_2512_02293_b200.device import DeviceProblem
    return DeviceProblem(P, opts)


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"cfg{c}")
def test_energy(cfg, cuda_ok):
    P, G = problem(cfg)
    dp = _dp(P, opts_of(G))
    e = dp.energy()[0]
    dp.close()
    ref = float(G["energy"])
    print(f"cfg{cfg} energy rel err {abs(e - ref) / ref:.2e}")
    assert abs(e - ref) <= TOL_COST * ref


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"cfg{c}")
def test_linearize(cfg, cuda_ok):
    P, G = problem(cfg)
    opts = opts_of(G)
    dp = _dp(P, opts)
    dp.linearize()
    cols = G["H_pd_cols"] if "H_pd_cols" in G else None
    H_pp, H_pd, H_dd, g_p, g_d = dp.export_normal_eq(with_hpd=cols is not None, hpd_cols=cols)
    dp.close()
    L = oracle.Layout(P, opts)
    H_imu, g_imu = oracle.vi_ba._imu_part(P, L)
    errs = {}
    errs["H_pp"], errs["H_pp_proj"] = mat_err(G, "H_pp", H_pp)
    # vision family: the reference's H_pp minus the (fp64, pinned) inertial part
    Gv = dict(G)
    if "H_pp" in G:
        Gv["H_pp"] = G["H_pp"] - H_imu
        Gv["H_pp_maxabs"] = np.abs(Gv["H_pp"]).max()
        Gv["H_pp_proj"] = G["H_pp_proj"] - H_imu @ golden_proj_vector(len(H_imu), 11)
        errs["H_vision"], _ = mat_err(Gv, "H_pp", H_pp - H_imu)
    else:
        Kb = len(H_imu) // 15
        Bi = H_imu.reshape(Kb, 15, Kb, 15)
        Gv["H_pp_diag"] = G["H_pp_diag"] - np.stack([Bi[k, :, k, :] for k in range(Kb)])
        Gv["H_pp_sub"] = G["H_pp_sub"] - np.stack([Bi[k + 1, :, k, :] for k in range(Kb - 1)])
        vis_max = max(np.abs(Gv["H_pp_diag"]).max(), np.abs(Gv["H_pp_sub"]).max(), np.abs(G["H_pp_oblk"]).max())
        Gv["H_pp_maxabs"] = vis_max
        Gv["H_pp_proj"] = G["H_pp_proj"] - H_imu @ golden_proj_vector(len(H_imu), 11)
        errs["H_vision"], _ = mat_err(Gv, "H_pp", H_pp - H_imu)
    errs["g_p"] = float(np.abs(g_p - G["g_p"]).max() / np.abs(G["g_p"]).max())
    gv_ref = G["g_p"] - g_imu
    errs["g_vision"] = float(np.abs((g_p - g_imu) - gv_ref).max() / np.abs(gv_ref).max())
    errs["H_dd"] = vec_err(G, "H_dd", H_dd)
    errs["g_d"] = vec_err(G, "g_d", g_d)
    if cols is not None:
        errs["H_pd"] = float(np.abs(H_pd - G["H_pd"]).max() / G["H_pd_maxabs"])
    print(f"cfg{cfg} linearize rel errs " + " ".join(f"{k}={v:.2e}" for k, v in errs.items()))
    for k, v in errs.items():
        assert v < TOL_H, (k, v)


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"cfg{c}")
def test_reduced_system(cfg, cuda_ok):
    P, G = problem(cfg)
    opts = opts_of(G)
    dp = _dp(P, opts)
    dp.linearize()
    Hr, gr = dp.export_reduced(opts["damping"])
    st = dp.stats()
    dp.close()
    e, ep = mat_err(G, "Hred", Hr)
    eg = float(np.abs(gr - G["gred"]).max() / np.abs(G["gred"]).max())
    print(f"cfg{cfg} H_red rel err {e:.2e} (proj {ep:.2e}), g_red {eg:.2e}")
    assert e < TOL_H and ep < TOL_H and eg < TOL_H
    assert st["fallbacks"] == 0


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"cfg{c}")
def test_step(cfg, cuda_ok):
    P, G = problem(cfg)
    opts = opts_of(G)
    dp = _dp(P, opts)
    dp.linearize()
    dx, dxd = dp.solve_step(opts["damping"])
    st = dp.stats()
    dp.close()
    ex = float(np.abs(dx - G["dx"]).max() / np.abs(G["dx"]).max())
    ed = vec_err(G, "dxd", dxd)
    print(f"cfg{cfg} step rel err dx={ex:.2e} dx_d={ed:.2e} (tensor-core solve: {st})")
    assert ex < TOL_DX and ed < TOL_DX
    assert st["fallbacks"] == 0


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"cfg{c}")
def test_solve(cfg, cuda_ok):
    P, G = problem(cfg)
    opts = opts_of(G)
    dp = _dp(copy.deepcopy(P), opts)
    rep = dp.solve()
    s = dp.download()
    st = dp.stats()
    dp.close()
    ref = G["meta"]["report"]
    c, cr = np.array(rep["cost_trajectory"]), np.array(ref["cost_trajectory"])
    print(f"cfg{cfg} solve: {rep['iterations']} it ({ref['iterations']}), {rep['termination']} "
          f"({ref['termination']}), cost rel errs {np.abs(c[:len(cr)] - cr[:len(c)]) / cr[:len(c)]}")
    assert rep["iterations"] == ref["iterations"]
    assert rep["termination"] == ref["termination"]
    assert len(c) == len(cr)
    assert np.all(np.abs(c - cr) <= TOL_COST * cr), (c, cr)
    assert rep["condition_warnings"] == ref["condition_warnings"]
    # final states: the accumulated update error relative to the total motion of the solve
    P0 = P
    for k in ("p", "v", "bg", "ba"):
        moved = np.abs(G["final_" + k] - P0[k]).max()
        err = np.abs(s[k] - G["final_" + k]).max()
        print(f"  final {k}: err {err:.2e} of motion {moved:.2e}")
        assert err <= TOL_DX * max(moved, 1e-12) + 1e-12, k
    dmoved = vec_err(G, "final_disp", s["disp"])
    print(f"  final disparities rel err {dmoved:.2e}")
    assert dmoved < TOL_DX
    assert st["fallbacks"] == 0


@pytest.mark.parametrize("cfg", [c for c in (1, 3) if c in CFGS], ids=lambda c: f"cfg{c}")
def test_gram_paths(cfg, cuda_ok, monkeypatch):
    """Both Schur Gram kernels at full size: the tcgen05 3xTF32 one (the default here, >= 256
    pixels per keyframe) and the exact fp64 DMMA one (VBA_GRAM=dmma; the default for small
    windows) meet the north_star tolerances against the reference, and agree with each other
    far inside them (the tf32 split keeps ~21 significant bits per factor)."""
    P, G = problem(cfg)
    opts = opts_of(G)
    out = {}
    for kind in ("tc", "dmma"):
        monkeypatch.setenv("VBA_GRAM", kind)
        dp = _dp(P, opts)
        assert dp.stats()["gram_tc"] == (kind == "tc")
        dp.linearize()
        Hr, gr = dp.export_reduced(opts["damping"])
        dx, dxd = dp.solve_step(opts["damping"])
        dp.close()
        e, _ = mat_err(G, "Hred", Hr)
        ex = float(np.abs(dx - G["dx"]).max() / np.abs(G["dx"]).max())
        ed = vec_err(G, "dxd", dxd)
        print(f"cfg{cfg} gram {kind}: H_red {e:.2e} dx {ex:.2e} dx_d {ed:.2e}")
        assert e < TOL_H and ex < TOL_DX and ed < TOL_DX
        out[kind] = (Hr, dx, dxd)
    (h1, x1, d1), (h0, x0, d0) = out["tc"], out["dmma"]
    dh = float(np.abs(h1 - h0).max() / np.abs(h0).max())
    dxx = float(np.abs(x1 - x0).max() / np.abs(x0).max())
    ddd = float(np.abs(d1 - d0).max() / np.abs(d0).max())
    print(f"cfg{cfg} tc vs dmma: H_red {dh:.2e} dx {dxx:.2e} dx_d {ddd:.2e}")
    assert dh < 1e-7 and dxx < 1e-6 and ddd < 1e-6
