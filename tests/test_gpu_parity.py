"""GPU parity: the CUDA path (libvba through the C ABI) against the reference.

Golden fixtures hold the reference's own outputs on fp32-representable inputs
(tests/golden/make_golden.py).  Tolerances follow BASELINE.json north_star,
graded per block family as SURVEY.md §8(c) prescribes:

* H and g: relative 1e-4 (max|Δ| / max|ref| within each family)
* pose / disparity updates: relative 1e-5
"""
import copy
import os

import numpy as np
import pytest

import oracle
from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

NAMES = golden_names()
TOL_H = 1e-4
TOL_DX = 1e-5


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    s = np.abs(b).max(initial=0.0)
    if s == 0.0:
        return float(np.abs(a).max(initial=0.0))
    return float(np.abs(a - b).max(initial=0.0) / s)


def _dp(P, opts):
    from paper_2512_02293_b200.device import DeviceProblem
    return DeviceProblem(P, opts)


@pytest.mark.parametrize("name", NAMES)
def test_energy(name, cuda_ok):
    P, out, opts = load_golden(name)
    dp = _dp(P, opts)
    e, ev, ei = dp.energy()
    ref = float(out["energy"])
    ev_ref, ei_ref = oracle.total_energy(P, parts=True)
    assert abs(e - ref) <= 1e-5 * ref + 1e-9
    assert abs(ei - ei_ref) <= 1e-10 * max(ei_ref, 1.0)       # IMU energy is fp64 end to end
    assert abs(ev - ev_ref) <= 1e-5 * max(ev_ref, 1e-6)


@pytest.mark.parametrize("name", NAMES)
def test_linearize(name, cuda_ok):
    P, out, opts = load_golden(name)
    dp = _dp(P, opts)
    dp.linearize()
    H_pp, H_pd, H_dd, g_p, g_d = dp.export_normal_eq()
    L = oracle.Layout(P, opts)
    H_imu, g_imu = oracle.vi_ba._imu_part(P, L)
    # inertial blocks (fp64 path) and vision blocks (fp32 per pixel) graded separately
    assert rel(H_pp, out["H_pp"]) < TOL_H
    if np.abs(out["H_pp"] - H_imu).max() > 1e-9 * np.abs(out["H_pp"]).max():
        assert rel(H_pp - H_imu, out["H_pp"] - H_imu) < TOL_H
        assert rel(g_p - g_imu, out["g_p"] - g_imu) < TOL_H
    assert rel(g_p, out["g_p"]) < TOL_H
    assert rel(H_dd, out["H_dd"]) < TOL_H
    assert rel(g_d, out["g_d"]) < TOL_H
    assert rel(H_pd, out["H_pd"]) < TOL_H


# Vision-only, pose-only 4-keyframe window: the metric scale is unobservable
# (frozen kf 0, no IMU), so H_red's scale direction is held only by the LM
# damping and the fp32 per-pixel linearisation noise (H itself within 3e-8) is
# amplified ~1e4 there (measured: dx 1.8e-4, dx_d 5.6e-4; the solve on the
# GPU's own linearisation agrees with fp64 to 1e-6).  Graded at 1e-3 and listed in DESIGN.md §6 as a known
# fp32 limitation.
ILL_CONDITIONED = {"win4_sdof6": 1e-3}


def tol_update(name, out, key):
    """1e-5 (north_star), or the reference's own sensitivity to sub-ulp fp32
    target noise when that is larger (golden 'cond_*', make_golden.py)."""
    return max(TOL_DX, 1.5 * float(out["cond_" + key]), ILL_CONDITIONED.get(name, 0.0))


@pytest.mark.parametrize("name", NAMES)
def test_solve_step(name, cuda_ok):
    P, out, opts = load_golden(name)
    dp = _dp(P, opts)
    dp.linearize()
    dx, dxd = dp.solve_step(opts["damping"])
    assert rel(dx, out["dx"]) < tol_update(name, out, "dx")
    assert rel(dxd, out["dxd"]) < tol_update(name, out, "dxd")


@pytest.mark.parametrize("name", ["win8_px30", "win5_gravity", "win6_frozen2", "cfg0_grid12x16"])
def test_dense_path_step(name, cuda_ok):
    """use_schur=False (solver.py:291-304) gives the reference's step too."""
    P, out, opts = load_golden(name)
    dp = _dp(P, dict(opts, use_schur=False))
    dp.linearize()
    dx, dxd = dp.solve_step(opts["damping"], use_schur=False)
    assert rel(dx, out["dx"]) < tol_update(name, out, "dx")
    assert rel(dxd, out["dxd"]) < tol_update(name, out, "dxd")


def test_baseline_shaped_step_within_north_star(cuda_ok):
    """The BASELINE-shaped fixture meets 1e-5 on both update families outright."""
    P, out, opts = load_golden("cfg0_grid12x16")
    dp = _dp(P, opts)
    dp.linearize()
    dx, dxd = dp.solve_step(opts["damping"])
    assert rel(dx, out["dx"]) < TOL_DX
    assert rel(dxd, out["dxd"]) < TOL_DX


@pytest.mark.parametrize("name", NAMES)
def test_solve_vi_ba(name, cuda_ok):
    P, out, opts = load_golden(name)
    dp = _dp(copy.deepcopy(P), opts)
    rep = dp.solve()
    ref = out["report"]
    s = dp.download()
    # costs agree while they are far above the fp32 energy floor (~1e-7 relative
    # noise of the per-pixel residuals times the initial cost)
    c, cr = rep["cost_trajectory"], ref["cost_trajectory"]
    floor = 1e-6 * cr[0]
    for k in range(min(len(cr), len(c))):
        if cr[k] < floor:
            break
        assert abs(c[k] - cr[k]) <= 1e-3 * cr[k], (k, c, cr)
    assert rep["iterations"] >= min(ref["iterations"], 2)
    # final states agree with the reference's converged states
    scale = 10.0 if name in ILL_CONDITIONED else 1.0   # unobservable scale: noise-driven drift
    assert np.abs(s["p"] - out["final_p"]).max() < 1e-5 * scale
    assert np.abs(s["v"] - out["final_v"]).max() < 1e-4 * scale
    assert np.abs(s["disp"] - out["final_disp"]).max() < 1e-4 * scale * np.abs(out["final_disp"]).max()


@pytest.mark.gpu
@pytest.mark.parametrize("n,cond", [(100, 1e3), (300, 1e6), (1000, 1e5), (1905, 1e7)])
def test_spd_solve_tensor_core_matches_fp64(cuda_ok, n, cond):
    """tcgen05 split-fp16 (3-product) Cholesky + fp64 refinement == fp64 solve (solver.py:287):
    refinement stops once a pass corrects x by <= 1e-5 max|x| and the geometric-tail bound of
    the error left is <= 1e-7 max|x| (k_tc_check)."""
    import torch
    from paper_2512_02293_b200 import _lib
    g = torch.Generator().manual_seed(n)
    Q, _ = torch.linalg.qr(torch.randn(n, n, generator=g, dtype=torch.float64))
    ev = torch.logspace(0, float(np.log10(cond)), n, dtype=torch.float64)
    d = torch.exp(torch.randn(n, generator=g, dtype=torch.float64) * 3.0)   # badly scaled rows, like H_red
    H = (d[:, None] * (Q * ev) @ Q.T * d[None, :])
    H = 0.5 * (H + H.T)
    b = torch.randn(n, generator=g, dtype=torch.float64)
    ref = torch.linalg.solve(H, b)
    Hd, bd = H.cuda(), b.cuda()
    x1, tc1 = _lib.spd_solve(Hd, bd, mode=1)
    x0, tc0 = _lib.spd_solve(Hd, bd, mode=0)
    assert not tc1
    assert tc0 or cond > 1e5          # ill-conditioned: tensor-core refinement may hand over to fp64
    e1 = ((x1.cpu() - ref).abs().max() / ref.abs().max()).item()
    e0 = ((x0.cpu() - ref).abs().max() / ref.abs().max()).item()
    assert e1 < 1e-9 * max(1.0, cond / 1e5), e1
    assert e0 < 1e-8 * max(1.0, cond / 1e5), e0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 8, 105, 165, 225, 232, 233])
def test_spd_solve_small_and_dag_fp64(cuda_ok, n, monkeypatch):
    """The one-CTA fp64 solve (n <= 232, vba_small.cu) and the fp64 tile DAG (VBA_CHOL=dag;
    n = 233 goes to the DAG either way) both reproduce np.linalg.solve (solver.py:287) on an
    ill-conditioned, badly scaled SPD system like H_red, including sizes that are not a
    multiple of the 8-column panel (identity padding)."""
    import torch
    from paper_2512_02293_b200 import _lib
    g = torch.Generator().manual_seed(1000 + n)
    Q, _ = torch.linalg.qr(torch.randn(n, n, generator=g, dtype=torch.float64))
    ev = torch.logspace(0, 6, n, dtype=torch.float64)
    d = torch.exp(torch.randn(n, generator=g, dtype=torch.float64) * 3.0)
    H = (d[:, None] * (Q * ev) @ Q.T * d[None, :])
    H = 0.5 * (H + H.T)
    b = torch.randn(n, generator=g, dtype=torch.float64)
    ref = torch.linalg.solve(H, b)
    x_small, _ = _lib.spd_solve(H.cuda(), b.cuda(), mode=1)
    monkeypatch.setenv("VBA_CHOL", "dag")
    x_dag, _ = _lib.spd_solve(H.cuda(), b.cuda(), mode=1)
    for x in (x_small, x_dag):
        err = ((x.cpu() - ref).abs().max() / ref.abs().max()).item()
        assert err < 1e-9, (n, err)
    # not positive definite: both report it (the reference's singular-system retry path)
    Hn = H.clone()
    Hn[n // 2, n // 2] = -abs(Hn[n // 2, n // 2])
    for mode_env in ("", "dag"):
        monkeypatch.setenv("VBA_CHOL", mode_env)
        with pytest.raises(Exception):
            _lib.spd_solve(Hn.cuda(), b.cuda(), mode=1)


@pytest.fixture
def force_tc(monkeypatch):
    """Force the tensor-core reduced solve (3xTF32 factor + fp64 refinement) on the
    small golden systems; by default it is only used from 32 Cholesky tiles up."""
    monkeypatch.setenv("VBA_CHOL", "tc")
    yield


def _stats(dp):
    import ctypes
    s = (ctypes.c_int64 * 4)()
    dp.lib.vba_stats(dp.ctx, s)
    return list(s)


@pytest.mark.parametrize("name", NAMES)
def test_solve_step_tensor_core(name, cuda_ok, force_tc):
    P, out, opts = load_golden(name)
    dp = _dp(P, opts)
    dp.linearize()
    dx, dxd = dp.solve_step(opts["damping"])
    st = _stats(dp)
    assert st[0] == 1 and st[2] >= 1, st                    # the tensor-core path ran
    assert rel(dx, out["dx"]) < tol_update(name, out, "dx")
    assert rel(dxd, out["dxd"]) < tol_update(name, out, "dxd")


@pytest.mark.parametrize("name", ["win8_px30", "cfg0_grid12x16", "win5_gravity"])
def test_solve_vi_ba_tensor_core(name, cuda_ok, force_tc):
    P, out, opts = load_golden(name)
    dp = _dp(copy.deepcopy(P), opts)
    rep = dp.solve()
    ref = out["report"]
    s = dp.download()
    c, cr = rep["cost_trajectory"], ref["cost_trajectory"]
    for k in range(min(len(cr), len(c))):
        if cr[k] < 1e-6 * cr[0]:
            break
        assert abs(c[k] - cr[k]) <= 1e-3 * cr[k], (k, c, cr)
    assert np.abs(s["p"] - out["final_p"]).max() < 1e-5
    assert _stats(dp)[1] == 0                                 # no fp64 fallback


def test_large_window_uses_tensor_core_solve_without_fallback(cuda_ok):
    """BASELINE config 3 (n_f = 1905 -> 15 tiles) forced onto the tensor-core solve: the
    solve converges (no fp64 fallback) and the step equals the fp64 DAG's to 1e-7
    (refinement stops at a 1e-6 relative correction, ~1e-9 error)."""
    import os
    from paper_2512_02293_b200.problem import pack_graph
    from paper_2512_02293_b200.workloads import make_workload
    P = pack_graph(make_workload(3))
    opts = {"max_iterations": 1}
    steps = {}
    for mode in ("fp64", "tc"):
        os.environ["VBA_CHOL"] = mode
        try:
            dp = _dp(copy.deepcopy(P), opts)
            dp.linearize()
            steps[mode] = dp.solve_step(1e-4)
            if mode == "tc":
                st = _stats(dp)
                assert st[0] == 1 and st[1] == 0 and st[2] >= 1, st
            dp.close()
        finally:
            os.environ.pop("VBA_CHOL", None)
    assert rel(steps["tc"][0], steps["fp64"][0]) < 1e-7
    assert rel(steps["tc"][1], steps["fp64"][1]) < 1e-7


def test_solve_windows_streams_bitwise_equal(cuda_ok):
    """The streaming entry point (device.solve_windows: window s+1 uploaded on a copy
    stream while window s is solved, inputs rebound with vba_bind_inputs) returns,
    for every window, exactly the state of a plain upload + solve of that window."""
    import torch
    from paper_2512_02293_b200.problem import pack_graph
    from paper_2512_02293_b200.workloads import make_workload
    P = pack_graph(make_workload(1))
    opts = {"max_iterations": 2}
    dp = _dp(copy.deepcopy(P), opts)
    H = dp.H
    base = {k: np.ascontiguousarray(v) for k, v in (("state", H.state), ("disp", H.disp), ("tgt", H.tgt),
                                                   ("w", H.w), ("imu", H.imu), ("grav", H.grav))}
    rng = np.random.default_rng(7)
    wins = []
    for s in range(3):   # three different windows: perturbed flow targets
        w = dict(base)
        w["tgt"] = (base["tgt"] + rng.normal(0.0, 0.2, base["tgt"].shape)).astype(base["tgt"].dtype)
        wins.append({k: torch.from_numpy(np.ascontiguousarray(v).reshape(-1)).pin_memory() for k, v in w.items()})
    outs = [(torch.empty(dp.d_state.shape, dtype=torch.float64).pin_memory(),
             torch.empty(dp.d_disp.shape, dtype=torch.float32).pin_memory()) for _ in wins]
    reps = dp.solve_windows(wins, outputs=outs)
    torch.cuda.synchronize()
    assert len(reps) == 3
    for s in range(3):
        ref = _dp(copy.deepcopy(P), opts)
        ref.d_tgt.copy_(wins[s]["tgt"].reshape(ref.d_tgt.shape))
        torch.cuda.synchronize()
        ref.load_state()
        r = ref.solve()
        ref.lib.vba_download(ref.ctx, ref._sptr())
        torch.cuda.synchronize()
        assert r["final_cost"] == reps[s]["final_cost"]
        assert torch.equal(ref.d_state.cpu(), outs[s][0])
        assert torch.equal(ref.d_disp.cpu(), outs[s][1])
        ref.close()
    dp.close()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_solve_is_bitwise_the_single_rank_solve(cuda_ok, world):
    """Edge-sharded LM solve (paper_2512_02293_b200.distributed) on BASELINE config 3 with
    2 / 3 ranks sharing this GPU (gloo, host-mediated gathers: no kernel waits on another
    rank's), against the one-rank solve: cost trajectory, states and every keyframe's
    disparities bitwise equal (tools/dist_check.py asserts it)."""
    import subprocess
    import sys
    from conftest import REPO
    port = 29400 + world + (os.getpid() % 500)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(REPO, "tools", "dist_check.py"), "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "dist_check ok" in r.stdout and "bitwise True" in r.stdout


def test_largest_config_properties(cuda_ok):
    """BASELINE config 4 at full size (n_f = 7665, 37.7 M edge-pixels), where the fp64
    oracle cannot run: size-independent properties of the path.
    * determinism: two linearise + reduced-solve passes give bitwise-equal steps;
    * the LM solve decreases the energy monotonically and reports exactly the energy the
      energy kernel returns for the final state;
    * no fp64 fallback of the tensor-core reduced solve."""
    from paper_2512_02293_b200.problem import pack_graph
    from paper_2512_02293_b200.workloads import CONFIGS, make_workload
    P = pack_graph(make_workload(4))
    opts = {"max_iterations": CONFIGS[4].iterations}
    dp = _dp(P, opts)
    dp.linearize()
    a = dp.solve_step(1e-4)
    dp.linearize()
    b = dp.solve_step(1e-4)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    dp.load_state()
    rep = dp.solve()
    traj = rep["cost_trajectory"]
    assert all(t1 <= t0 for t0, t1 in zip(traj, traj[1:]))
    assert rep["final_cost"] < rep["initial_cost"]
    assert abs(dp.energy()[0] - rep["final_cost"]) <= 1e-12 * rep["final_cost"]
    st = _stats(dp)
    assert st[1] == 0, st   # no fp64 fallbacks
    dp.close()


def test_spd_solve_at_tensor_core_residency_limit(cuda_ok):
    """n_free = 148 * 128 = 18944: the largest system the tensor-core path takes -- one
    cooperative CTA per SM for the 148-tile DAG (11 026 lower tiles) and for each triangular
    sweep (no helpers) -- against the fp64 solve."""
    import torch
    from paper_2512_02293_b200 import _lib
    n = 148 * 128
    g = torch.Generator(device="cuda").manual_seed(6)
    A = torch.randn(n, 64, generator=g, device="cuda", dtype=torch.float64)
    H = A @ A.T / 64.0
    H.diagonal().add_(1.0 + torch.rand(n, generator=g, device="cuda", dtype=torch.float64))
    b = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
    x, used_tc = _lib.spd_solve(H, b, mode=0)
    assert used_tc
    ref = torch.linalg.solve(H, b)
    err = ((x - ref).abs().max() / ref.abs().max()).item()
    print(f"n={n}: tensor-core solve rel err {err:.2e}")
    assert err < 1e-7


def test_spd_solve_beyond_tensor_core_residency(cuda_ok):
    """n_free > 148 * 128 = 18944: the tensor-core solve's triangular sweeps cannot keep one CTA
    per row tile resident, so chol_tc_solve declines (returns before refining) and the system
    is solved on the fp64 tile DAG -- never an unsolved zero step."""
    import torch
    from paper_2512_02293_b200 import _lib
    n = 19200
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(n, 64, generator=g, device="cuda", dtype=torch.float64)
    H = A @ A.T / 64.0
    H.diagonal().add_(1.0 + torch.rand(n, generator=g, device="cuda", dtype=torch.float64))
    b = torch.randn(n, generator=g, device="cuda", dtype=torch.float64)
    x, used_tc = _lib.spd_solve(H, b, mode=0)
    assert not used_tc
    ref = torch.linalg.solve(H, b)
    err = ((x - ref).abs().max() / ref.abs().max()).item()
    print(f"n={n}: fp64 DAG solve rel err {err:.2e}")
    assert err < 1e-9


def _high_degree_graph(degrees, seed=7):
    """Config 1 on a 24x32 grid with the out-edges of some sources duplicated (re-weighted) up
    to the requested out-degrees: the reference accepts repeated keyframe pairs
    (solver.py:62-73), and global graphs reach such degrees."""
    from paper_2512_02293_b200 import types as T
    from paper_2512_02293_b200.workloads import make_workload
    g = make_workload(1, grid=(24, 32))
    rng = np.random.default_rng(seed)
    edges = list(g.vision_edges)
    for src, deg in degrees.items():
        own = [e for e in edges if e.i == src]
        for t in range(deg - len(own)):
            e = own[t % len(own)]
            w = (e.weights * rng.uniform(0.5, 1.5, e.weights.shape)).astype(np.float32).astype(float)
            edges.append(T.VisionEdge(e.i, e.j, e.pixels, e.targets, w))
    edges.sort(key=lambda e: e.i)
    g.vision_edges = edges
    return g


@pytest.mark.gpu
def test_high_out_degree_sources(cuda_ok):
    """Sources with 40 and 63 out-edges (beyond one Gram CTA's 31: the DMMA Gram in unit slices,
    the fill-in transform reading its record in place) against the fp64 oracle: reduced system,
    step and a full solve; 64 out-edges are refused with VBA_E_UNSUPPORTED."""
    from paper_2512_02293_b200.device import DeviceProblem
    from paper_2512_02293_b200.problem import pack_graph
    from oracle import vi_ba as O
    g = _high_degree_graph({5: 40, 9: 63})
    P = pack_graph(g)
    opts = {"max_iterations": 3, "frozen_keyframes": (0,)}
    o = dict(O.DEFAULT_OPTS)
    o.update(opts)
    L = O.Layout(P, o)
    lin = O.linearize_sparse(P, L)
    Hr_ref, gr_ref, _ = O.reduced_system_sparse(L, o, *lin, o["damping"])
    free = L.free_mask()
    dx_ref, dxd_ref = O.solve_step_sparse(L, o, *lin, o["damping"])
    dp = DeviceProblem(P, opts)
    assert dp.stats()["gram_tc"] == 0
    dp.linearize()
    Hr, gr = dp.export_reduced(o["damping"])
    dx, dxd = dp.solve_step(o["damping"])
    eh = np.abs(Hr - Hr_ref[np.ix_(free, free)]).max() / np.abs(Hr_ref).max()
    eg = np.abs(gr - gr_ref[free]).max() / np.abs(gr_ref).max()
    ex = np.abs(dx - dx_ref).max() / np.abs(dx_ref).max()
    ed = np.abs(dxd - dxd_ref).max() / np.abs(dxd_ref).max()
    print(f"out-degree 40/63: H_red {eh:.1e} g_red {eg:.1e} dx {ex:.1e} dx_d {ed:.1e}")
    assert eh < 1e-4 and eg < 1e-4 and ex < 1e-5 and ed < 1e-5
    rep = dp.solve()
    ref = O.solve_vi_ba(copy.deepcopy(P), opts, sparse=True)
    print("costs", rep["cost_trajectory"], ref["cost_trajectory"])
    assert rep["iterations"] == ref["iterations"] and rep["termination"] == ref["termination"]
    assert np.allclose(rep["cost_trajectory"], ref["cost_trajectory"], rtol=1e-6)
    dp.close()
    from paper_2512_02293_b200 import _lib
    with pytest.raises(_lib.VbaError) as ei:
        DeviceProblem(pack_graph(_high_degree_graph({9: 64})), opts)
    assert ei.value.code == _lib.VBA_E_UNSUPPORTED
