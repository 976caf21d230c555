"""Goldens at the BASELINE configs (build container only; the GPU box reads the npz).

For every BASELINE.json config the seeded window of
``paper_2512_02293_b200.workloads.make_workload(cfg)`` is solved on the CPU and
the outputs the GPU path must reproduce are stored in ``tests/golden/bcfg<cfg>.npz``:

* cfg 0, 1, 2: the REFERENCE itself (vislam imported read-only from
  /root/reference/pkg/src): ``total_energy``, ``_linearize``, the Schur system
  of ``_solve_step`` (harness restatement of solver.py:276-285 on the
  reference's own H_pp/H_pd), ``_solve_step`` dx / dx_d at λ = opts.damping,
  and ``solve_vi_ba`` with the BASELINE iteration count (report + final states);
* cfg 3: the reference as well (≈7 min, 17 GB: dense H_pd of 6 GB);
* cfg 4: the reference cannot run (dense H_pd alone is 96.6 GB), so the pinned
  per-keyframe sparse restatement ``oracle.vi_ba`` (linearize_sparse,
  reduced_system_sparse, solve_step_sparse, solve_vi_ba(sparse=True)) is used;
  it is pinned to the reference at cfg 0/1/3 by tests/test_oracle_golden.py.

The inputs are NOT stored: the test regenerates them with ``make_workload`` and
checks ``input_hash`` (sha256 of the packed arrays) first, so a generator drift
fails loudly instead of comparing different problems.  Large outputs are
stored sampled (conftest.golden_* helpers document the scheme):

* per-pixel vectors (H_dd, g_d, dx_d, final disparities): full up to 65 536
  entries, else 32 768 seeded indices plus the full max|ref|;
* pose-space matrices (H_pp, H_red): full up to 256 columns, else every
  diagonal and sub-diagonal sdof×sdof block plus up to 1500 other non-zero
  lower blocks (their pose 6×6 part: everything else in them is exactly zero,
  asserted here), plus the product with a seeded vector;
* the coupling H_pd: 256 seeded disparity columns per keyframe (cfg 0-2; 4 of them at cfg 3).

Run:  python tests/golden/make_config_golden.py 0 1 2 3 4
"""

from __future__ import annotations

import copy
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from conftest import (GOLD_FULL_MAT, GOLD_FULL_VEC, GOLD_OTHER_BLOCKS, GOLD_VEC_SAMPLES,  # noqa: E402
                      golden_proj_vector, golden_vec_indices, packed_hash)

from paper_2512_02293_b200.problem import pack_graph  # noqa: E402
from paper_2512_02293_b200.workloads import CONFIGS, make_workload  # noqa: E402

OPT_KEYS = ("max_iterations", "damping", "damping_up", "damping_down", "rel_decrease_tol", "step_tol",
            "max_damping", "frozen_keyframes", "optimize_gravity", "optimize_velocity_bias", "use_schur", "ridge")


def vec_entry(out, name, v, seed):
    v = np.asarray(v, np.float64)
    out[name + "_n"] = np.array(len(v))
    out[name + "_maxabs"] = np.array(np.abs(v).max(initial=0.0))
    if len(v) <= GOLD_FULL_VEC:
        out[name] = v
    else:
        idx = golden_vec_indices(len(v), seed)
        out[name + "_idx"] = idx
        out[name] = v[idx]


def mat_entry(out, name, M, sdof, K_blocks, seed):
    """Pose-space symmetric matrix M (n x n, n = K_blocks*sdof [+ gravity])."""
    M = np.asarray(M, np.float64)
    n = M.shape[0]
    out[name + "_n"] = np.array(n)
    out[name + "_maxabs"] = np.array(np.abs(M).max(initial=0.0))
    v = golden_proj_vector(n, seed)
    out[name + "_proj"] = M @ v
    if n <= GOLD_FULL_MAT:
        out[name] = M
        return
    assert n == K_blocks * sdof, "gravity columns only occur in the small windows"
    B = M.reshape(K_blocks, sdof, K_blocks, sdof).transpose(0, 2, 1, 3)
    nz = np.abs(B).max(axis=(2, 3)) > 0
    diag = np.stack([B[k, k] for k in range(K_blocks)])
    sub = np.stack([B[k + 1, k] for k in range(K_blocks - 1)])
    others = [(a, b) for a in range(K_blocks) for b in range(a - 1) if nz[a, b]]
    rng = np.random.default_rng(seed + 7)
    if len(others) > GOLD_OTHER_BLOCKS:
        pick = np.sort(rng.choice(len(others), GOLD_OTHER_BLOCKS, replace=False))
        others = [others[k] for k in pick]
    ob = np.stack([B[a, b] for a, b in others]) if others else np.zeros((0, sdof, sdof))
    # vision-only couplings: only the pose (rot, trans) 6x6 part can be non-zero
    assert np.all(ob[:, 6:, :] == 0) and np.all(ob[:, :, 6:] == 0)
    out[name + "_diag"] = diag
    out[name + "_sub"] = sub
    out[name + "_oidx"] = np.array(others, np.int32).reshape(-1, 2)
    out[name + "_oblk"] = ob[:, :6, :6]


def free_keyframe_blocks(frozen_mask):
    return int((~frozen_mask).sum())


def reduced_from_dense(H_pp, H_pd, H_dd, g_p, g_d, free, lam, ridge):
    """solver.py:272-285 on the reference's own dense outputs (harness restatement)."""
    Hf = H_pp[np.ix_(free, free)].copy()
    idx = np.arange(Hf.shape[0])
    Hf[idx, idx] = np.diag(Hf) * (1.0 + lam) + ridge
    Hfd = H_pd[free]
    inv = 1.0 / (H_dd * (1.0 + lam) + ridge)
    Hred = Hf - (Hfd * inv) @ Hfd.T
    gred = g_p[free] - Hfd @ (inv * g_d)
    return Hred, gred


def run_reference(cfg, g, opts_ref, iters):
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, os.path.join(HERE))
    from make_golden import to_reference_graph
    from vislam import solver as S

    rg = to_reference_graph(g)
    o = S.SolveOptions(**{k: (tuple(v) if k == "frozen_keyframes" else v) for k, v in opts_ref.items()})
    lay = S._Layout(rg, o)
    t = time.time()
    energy = S.total_energy(rg)
    H_pp, H_pd, H_dd, g_p, g_d = S._linearize(rg, lay)
    print(f"  reference linearize {time.time() - t:.1f} s", flush=True)
    free = lay.free_mask()
    Hred, gred = reduced_from_dense(H_pp, H_pd, H_dd, g_p, g_d, free, o.damping, o.ridge)
    dx, dxd = S._solve_step(lay, H_pp, H_pd, H_dd, g_p, g_d, o.damping, True)
    res = dict(energy=energy, H_pp=H_pp, H_pd=H_pd, H_dd=H_dd, g_p=g_p, g_d=g_d, Hred=Hred, gred=gred,
               dx=dx, dxd=dxd, free=free)
    del H_pd
    rg2 = to_reference_graph(g)
    o2 = copy.deepcopy(o)
    o2.max_iterations = iters
    t = time.time()
    rep = S.solve_vi_ba(rg2, o2)
    print(f"  reference solve_vi_ba {time.time() - t:.1f} s", flush=True)
    res["report"] = dict(iterations=rep.iterations, initial_cost=rep.initial_cost, final_cost=rep.final_cost,
                         cost_trajectory=list(rep.cost_trajectory), termination=rep.termination,
                         condition_warnings=list(rep.condition_warnings))
    res["final"] = pack_graph(rg2)
    return res


def run_oracle(P, opts, iters):
    import oracle
    from oracle import vi_ba as V

    L = oracle.Layout(P, opts)
    t = time.time()
    energy = oracle.total_energy(P)
    H_pp, Hpd, H_dd, g_p, g_d = oracle.linearize_sparse(P, L)
    print(f"  oracle linearize {time.time() - t:.1f} s", flush=True)
    free = L.free_mask()
    H, g, _ = V.reduced_system_sparse(L, opts, H_pp, Hpd, H_dd, g_p, g_d, opts["damping"])
    Hred, gred = H[np.ix_(free, free)], g[free]
    dx, dxd = oracle.solve_step_sparse(L, opts, H_pp, Hpd, H_dd, g_p, g_d, opts["damping"])
    res = dict(energy=energy, H_pp=H_pp, H_pd=None, H_dd=H_dd, g_p=g_p, g_d=g_d, Hred=Hred, gred=gred,
               dx=dx, dxd=dxd, free=free)
    Q = copy.deepcopy(P)
    t = time.time()
    rep = oracle.solve_vi_ba(Q, dict(opts, max_iterations=iters), sparse=True)
    print(f"  oracle solve_vi_ba {time.time() - t:.1f} s", flush=True)
    res["report"] = rep
    res["final"] = Q
    return res


def main(cfgs):
    for cfg in cfgs:
        spec = CONFIGS[cfg]
        t0 = time.time()
        g = make_workload(cfg)
        P = pack_graph(g)
        opts = dict(max_iterations=spec.iterations, damping=1e-4, damping_up=10.0, damping_down=0.5,
                    rel_decrease_tol=1e-8, step_tol=1e-10, max_damping=1e8, frozen_keyframes=(0,),
                    optimize_gravity=False, optimize_velocity_bias=True, use_schur=True, ridge=1e-10)
        source = "oracle" if cfg == 4 else "reference"
        print(f"cfg{cfg}: {len(P['kid'])} kf, {len(P['ei'])} edges, {len(P['tgt'])} edge-px ({source})", flush=True)
        res = run_oracle(P, opts, spec.iterations) if source == "oracle" else run_reference(cfg, g, opts,
                                                                                          spec.iterations)
        K = len(P["kid"])
        sdof = 15
        out = {}
        meta = dict(cfg=cfg, source=source, input_hash=packed_hash(P), opts=dict(opts, frozen_keyframes=[0]),
                    K=K, sdof=sdof, n_disp=int(P["doff"][-1]), npv=K * sdof,
                    report=res["report"])
        out["energy"] = np.array(res["energy"])
        mat_entry(out, "H_pp", res["H_pp"], sdof, K, 11)
        mat_entry(out, "Hred", res["Hred"], sdof, int(res["free"].sum()) // sdof, 12)
        out["g_p"] = np.asarray(res["g_p"])
        out["gred"] = np.asarray(res["gred"])
        out["dx"] = np.asarray(res["dx"])
        vec_entry(out, "H_dd", res["H_dd"], 21)
        vec_entry(out, "g_d", res["g_d"], 22)
        vec_entry(out, "dxd", res["dxd"], 23)
        F = res["final"]
        for k in ("q", "p", "v", "bg", "ba", "grav_q"):
            out["final_" + k] = np.asarray(F[k])
        vec_entry(out, "final_disp", F["disp"], 24)
        if res["H_pd"] is not None:
            doff = P["doff"]
            rng = np.random.default_rng(31)
            cols = np.concatenate([np.sort(rng.choice(np.arange(doff[k], doff[k + 1]), 256, replace=False))
                                   for k in range(K)])
            if K * 15 > GOLD_FULL_MAT:     # large windows: 4 of those columns per keyframe (size)
                cols = cols.reshape(K, 256)[:, ::64].ravel()
            out["H_pd_cols"] = cols.astype(np.int64)
            out["H_pd"] = np.asarray(res["H_pd"][:, cols])
            out["H_pd_maxabs"] = np.array(np.abs(res["H_pd"]).max())
        out["meta"] = np.array(json.dumps(meta))
        path = os.path.join(HERE, f"bcfg{cfg}.npz")
        np.savez_compressed(path, **out)
        rep = res["report"]
        print(f"cfg{cfg}: energy {float(res['energy']):.9e}, {rep['iterations']} it, {rep['termination']}, "
              f"costs {rep['cost_trajectory']} -> {os.path.getsize(path) / 1e6:.2f} MB in {time.time() - t0:.0f} s",
              flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [0, 1, 2])
