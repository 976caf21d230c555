"""Drop-in replacement for ``vislam.loopclosure.solve_pgba`` (Sim(3) pose-graph BA) on the GPU.

Reference: /root/reference/pkg/src/vislam/loopclosure.py:378-574 (``total_pg_energy``,
``_PgLayout``, ``_linearize_pg``, ``_pg_apply``, ``solve_pgba``), with the factors
``sim3_vision_residual`` (loopclosure.py:225-307) and ``relative_pose_residual``
(residuals.py:364-380), and the shared damped Schur step ``solver._solve_step``
(loopclosure.py:27,534).

``solve_pgba(graph, opts=None) -> (SolveReport, LoopCorrection)`` has the reference's
semantics: the earliest keyframe is the gauge and is never touched; every other node's
Sim(3) state and the loop-source disparities are replaced in place by new objects;
``ValueError`` for a graph without loops or with a disconnected chain,
``RuntimeError`` for a non-finite initial energy.  The graph is read duck-typed
(reference classes or ``paper_2512_02293_b200.types``).  All arithmetic runs in
libvba (include/vba.h, ``vba_pg_*``; csrc/vba_pgba.cu).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .types import SolveOptions, SolveReport

SIM3_DOF = 7
PG_REL_REC = L.PG_REL_REC   # doubles per relative edge record (VBA_PG_REL_REC)


def pack_pose_graph(graph) -> dict:
    """Packed arrays of a PoseGraph (the layout oracle/pgba.py documents).

    Node order is the graph's (sorted by kid); relative edges are the loops without a
    vision edge (graph.loops order) followed by the chain (graph.chain order) --
    the reference's energy / linearisation order (loopclosure.py:378-390, 445-473)."""
    if not graph.loops:
        raise ValueError("pose graph has no loop edges")                   # loopclosure.py:510-511
    if len(graph.nodes) > 1 and not graph.chain:
        raise ValueError("pose graph chain is disconnected")               # :512-513
    nodes = list(graph.nodes)
    K = len(nodes)
    index = {n.kid: k for k, n in enumerate(nodes)}
    P = {}
    P["kid"] = np.array([n.kid for n in nodes], dtype=np.int64)
    P["sq"] = np.array([np.asarray(n.state.rotation.q, float) for n in nodes]).reshape(K, 4)
    P["st"] = np.array([np.asarray(n.state.translation, float) for n in nodes]).reshape(K, 3)
    P["ss"] = np.array([float(n.state.scale) for n in nodes])
    P["ts"] = np.array([float(getattr(n, "timestamp", 0.0)) for n in nodes])
    vis = [lp for lp in graph.loops if lp.vision is not None]
    sources = {lp.vision.i for lp in vis}
    counts = np.array([len(n.disparities) if n.kid in sources else 0 for n in nodes], dtype=np.int64)
    P["doff"] = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    src_nodes = [n for n in nodes if n.kid in sources]
    P["pix"] = (np.concatenate([np.asarray(n.pixels, float).reshape(-1, 2) for n in src_nodes])
                if src_nodes else np.zeros((0, 2)))
    P["disp"] = (np.concatenate([np.asarray(n.disparities, float).reshape(-1) for n in src_nodes])
                 if src_nodes else np.zeros(0))
    if len(P["disp"]) and P["disp"].min() <= 0.0:
        raise ValueError("disparities must be strictly positive")
    P["vi"] = np.array([index[lp.i] for lp in vis], dtype=np.int64)
    P["vj"] = np.array([index[lp.j] for lp in vis], dtype=np.int64)
    rows = np.array([len(lp.vision.pixels) for lp in vis], dtype=np.int64)
    for lp, n in zip(vis, rows):
        if n != counts[index[lp.i]]:
            raise ValueError("disparity length must match edge pixel list")
    P["veoff"] = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    cat = (lambda xs: np.concatenate([np.asarray(x, float).reshape(-1, 2) for x in xs]) if xs else np.zeros((0, 2)))
    P["vpix"] = cat([lp.vision.pixels for lp in vis])
    P["vtgt"] = cat([lp.vision.targets for lp in vis])
    P["vw"] = cat([lp.vision.weights for lp in vis])
    rel = [lp.relative for lp in graph.loops if lp.vision is None] + list(graph.chain)
    R = len(rel)
    P["ri"] = np.array([index[e.i] for e in rel], dtype=np.int64)
    P["rj"] = np.array([index[e.j] for e in rel], dtype=np.int64)
    P["rq"] = np.array([np.asarray(e.measurement.rotation.q, float) for e in rel]).reshape(R, 4)
    P["rt"] = np.array([np.asarray(e.measurement.translation, float) for e in rel]).reshape(R, 3)
    P["rs"] = np.array([float(e.measurement.scale) for e in rel])
    P["rinfo"] = np.array([np.asarray(e.information, float) for e in rel]).reshape(R, 7, 7)
    P["n_loops"] = len(graph.loops)
    k = graph.intrinsics
    P["intr"] = (np.array([k.fx, k.fy, k.cx, k.cy], dtype=float) if k is not None else np.array([1.0, 1.0, 0, 0]))
    T = getattr(graph, "T_cb", None)
    P["has_Tcb"] = T is not None
    P["Tcb"] = (np.concatenate([np.asarray(T.rotation.q, float), np.asarray(T.translation, float)])
                if T is not None else np.array([1.0, 0, 0, 0, 0, 0, 0]))
    return P


def _sorted_by_source(P):
    """Loop vision edges stably sorted by source node (the device plans per source)."""
    vi = np.asarray(P["vi"], np.int64)
    order = np.argsort(vi, kind="stable")
    if np.array_equal(order, np.arange(len(vi))):
        return P
    Q = dict(P)
    eo = np.asarray(P["veoff"], np.int64)
    segs = [(eo[v], eo[v + 1]) for v in order]
    Q["vi"], Q["vj"] = vi[order], np.asarray(P["vj"])[order]
    Q["veoff"] = np.concatenate([[0], np.cumsum([b - a for a, b in segs])]).astype(np.int64)
    for k in ("vpix", "vtgt", "vw"):
        Q[k] = np.concatenate([P[k][a:b] for a, b in segs])
    return Q


class DevicePoseGraph:
    """One pose graph resident on the current CUDA device (vba_pg_* C ABI)."""

    def __init__(self, P, opts: dict, stream=None):
        import torch
        if not L.cuda_available():
            raise RuntimeError("paper_2512_02293_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
        self.lib = L.load()
        self.P = P
        self.opts = dict(opts)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        P = _sorted_by_source(P)
        self.P = P
        K, V, R = len(P["kid"]), len(P["vi"]), len(P["ri"])
        nd = int(P["doff"][-1])
        nr = int(P["veoff"][-1])
        self.K, self.V, self.R, self.n_disp = K, V, R, nd
        doff = np.asarray(P["doff"], np.int64)
        npix = np.diff(doff).astype(np.int32)
        for v in range(V):
            r0, r1 = int(P["veoff"][v]), int(P["veoff"][v + 1])
            i = int(P["vi"][v])
            if not np.array_equal(P["vpix"][r0:r1], P["pix"][doff[i]:doff[i + 1]]):
                raise ValueError("loop vision rows must align with the source pixel snapshot")
        if len(P["vw"]) and np.min(P["vw"]) < 0:
            raise ValueError("weights must be non-negative")
        state = np.concatenate([P["sq"], P["st"], np.asarray(P["ss"])[:, None]], axis=1).reshape(K, 8)
        rel = np.zeros((R, PG_REL_REC))
        if R:
            rel[:, 0:4] = P["rq"]
            rel[:, 4:7] = P["rt"]
            rel[:, 7] = P["rs"]
            rel[:, 8:57] = np.asarray(P["rinfo"]).reshape(R, 49)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).to(dev)  # noqa: E731
        self.d_state = t(state)
        self.d_disp = t(P["disp"]) if nd else torch.zeros(1, dtype=torch.float64, device=dev)
        self.d_pix = t(P["pix"]) if nd else torch.zeros(2, dtype=torch.float64, device=dev)
        self.d_tgt = t(P["vtgt"]) if nr else torch.zeros(2, dtype=torch.float64, device=dev)
        self.d_w = t(P["vw"]) if nr else torch.zeros(2, dtype=torch.float64, device=dev)
        self.d_rel = t(rel) if R else torch.zeros(PG_REL_REC, dtype=torch.float64, device=dev)
        self._h = [np.ascontiguousarray(a) for a in (
            doff, npix, np.asarray(P["vi"], np.int32), np.asarray(P["vj"], np.int32),
            np.asarray(P["veoff"], np.int64), np.asarray(P["ri"], np.int32), np.asarray(P["rj"], np.int32))]
        p = L.VbaPgProblem()
        p.n_nodes, p.n_vis, p.n_rel = K, V, R
        p.n_disp, p.n_rows = nd, nr
        p.fx, p.fy, p.cx, p.cy = (float(x) for x in P["intr"])
        p.has_Tcb = int(bool(P["has_Tcb"]))
        for k in range(7):
            p.Tcb[k] = float(P["Tcb"][k])
        p.state, p.disp, p.pix, p.tgt, p.wts, p.rel = (x.data_ptr() for x in (
            self.d_state, self.d_disp, self.d_pix, self.d_tgt, self.d_w, self.d_rel))
        (p.h_doff, p.h_npix, p.h_vis_i, p.h_vis_j, p.h_voff, p.h_rel_i, p.h_rel_j) = (a.ctypes.data for a in self._h)
        o = L.VbaOptions()
        o.max_iterations = int(self.opts.get("max_iterations", 10))
        o.damping = float(self.opts.get("damping", 1e-4))
        o.damping_up = float(self.opts.get("damping_up", 10.0))
        o.damping_down = float(self.opts.get("damping_down", 0.5))
        o.rel_decrease_tol = float(self.opts.get("rel_decrease_tol", 1e-8))
        o.step_tol = float(self.opts.get("step_tol", 1e-10))
        o.max_damping = float(self.opts.get("max_damping", 1e8))
        o.optimize_gravity = 0
        o.optimize_velocity_bias = 0
        o.use_schur = int(bool(self.opts.get("use_schur", True)))
        o.ridge = float(self.opts.get("ridge", 1e-10))
        self._p, self._o = p, o
        ctx = C.c_void_p()
        L.check(self.lib.vba_pg_create(C.byref(ctx), C.byref(p), C.byref(o), self._sptr()))
        self.ctx = ctx

    def _sptr(self):
        return C.c_void_p(self.stream.cuda_stream)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.vba_pg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def energy(self):
        e = C.c_double()
        L.check(self.lib.vba_pg_energy(self.ctx, self._sptr(), C.byref(e)))
        return e.value

    def linearize(self):
        L.check(self.lib.vba_pg_linearize(self.ctx, self._sptr()))

    def export_normal_eq(self, hpd_cols=None):
        """(H_pp, H_pd[:, cols], H_dd, g_p, g_d) in the reference layout (loopclosure.py:425-475)."""
        import torch
        dev = self.device
        npv, nd = self.K * SIM3_DOF, self.n_disp
        Hpp = torch.empty((npv, npv), dtype=torch.float64, device=dev)
        gp = torch.empty(npv, dtype=torch.float64, device=dev)
        Hpd = torch.empty((npv, max(nd, 1)), dtype=torch.float64, device=dev)
        Hdd = torch.empty(max(nd, 1), dtype=torch.float64, device=dev)
        gd = torch.empty(max(nd, 1), dtype=torch.float64, device=dev)
        L.check(self.lib.vba_pg_export_normal_eq(self.ctx, self._sptr(), Hpp.data_ptr(), gp.data_ptr(), Hpd.data_ptr(),
                                                 Hdd.data_ptr(), gd.data_ptr()))
        Hpd = Hpd[:, :nd] if hpd_cols is None else Hpd[:, torch.as_tensor(hpd_cols, device=dev)]
        return (Hpp.cpu().numpy(), Hpd.cpu().numpy(), Hdd[:nd].cpu().numpy(), gp.cpu().numpy(),
                gd[:nd].cpu().numpy())

    def solve_step(self, lam, use_schur=True):
        """_solve_step on the pose graph (loopclosure.py:534): (dx_full [7K], dx_d [n_disp])."""
        import torch
        rc = self.lib.vba_pg_solve_step(self.ctx, self._sptr(), float(lam), int(bool(use_schur)))
        if rc == L.VBA_E_NOT_SPD:   # solver.py:287-289 / 300-303
            dense = not use_schur and self.n_disp > 0
            raise RuntimeError("singular full system" if dense else "singular reduced pose system")
        L.check(rc)
        dx = torch.empty(self.K * SIM3_DOF, dtype=torch.float64, device=self.device)
        dxd = torch.empty(max(self.n_disp, 1), dtype=torch.float64, device=self.device)
        L.check(self.lib.vba_pg_export_step(self.ctx, self._sptr(), dx.data_ptr(), dxd.data_ptr()))
        return dx.cpu().numpy(), dxd[:self.n_disp].cpu().numpy()

    def solve(self):
        cap = 4 * int(self._o.max_iterations) + 8
        traj = (C.c_double * cap)()
        rep = L.VbaReport()
        rc = self.lib.vba_pg_solve(self.ctx, self._sptr(), C.byref(rep), traj, cap)
        if rc == L.VBA_E_NONFINITE:
            raise RuntimeError("pose-graph energy is not finite")          # loopclosure.py:520-521
        L.check(rc)
        msg = ("singular full system" if not self._o.use_schur and self.n_disp > 0
               else "singular reduced pose system")
        term = {0: "max_iterations", 1: "converged", 2: "no_decrease_at_max_damping"}.get(
            rep.termination, "singular: " + msg)
        return dict(iterations=rep.iterations, initial_cost=rep.initial_cost, final_cost=rep.final_cost,
                    cost_trajectory=[traj[i] for i in range(min(rep.n_costs, cap))], termination=term,
                    condition_warnings=[msg] * rep.n_warnings, trials=rep.trials)

    def download(self):
        """(states [K,8] = q wxyz, t, scale; disparities [n_disp] in the packed order)."""
        L.check(self.lib.vba_pg_download(self.ctx, self._sptr()))
        self.stream.synchronize()
        s = self.d_state.cpu().numpy().reshape(self.K, 8)
        d = self.d_disp.cpu().numpy()[:self.n_disp]
        return s, d


def _correction(graph, before):
    """loopclosure.py:577-589 with the graph's own classes."""
    entries = {}
    stamp = 0.0
    for node in graph.nodes:
        old = before[node.kid]
        E = _cls(graph, "CorrectionEntry")
        entries[node.kid] = E(kid=node.kid, old_pose=old.pose(), new_pose=node.state.pose(),
                              scale_change=node.state.scale / old.scale)
        stamp = max(stamp, getattr(node, "timestamp", 0.0))
    return _cls(graph, "LoopCorrection")(entries, stamp)


def _cls(graph, name):
    """The caller's own class ``name`` (from the module defining its PoseGraph), else ours."""
    import sys
    from . import types as T
    mod = sys.modules.get(type(graph).__module__)
    return getattr(mod, name, None) or getattr(T, name)


def solve_pgba(graph, opts=None):
    """loopclosure.py:502-574 on the GPU; returns (SolveReport, LoopCorrection)."""
    if opts is None:
        opts = SolveOptions()
    P = pack_pose_graph(graph)
    before = {n.kid: n.state.copy() for n in graph.nodes}
    from .problem import _rotation_exact, options_dict
    dp = DevicePoseGraph(P, options_dict(opts))
    try:
        rep = dp.solve()
        if rep["iterations"] > 0:
            s, d = dp.download()
            doff = P["doff"]
            for k, node in enumerate(graph.nodes):
                if k > 0:    # the earliest keyframe is the gauge (loopclosure.py:403, 491)
                    st = node.state
                    node.state = type(st)(_rotation_exact(type(st.rotation), s[k, 0:4]), s[k, 4:7].copy(),
                                          float(s[k, 7]))
                if doff[k + 1] > doff[k]:
                    node.disparities = d[doff[k]:doff[k + 1]].copy()
    finally:
        dp.close()
    report = SolveReport(rep["iterations"], rep["initial_cost"], rep["final_cost"], rep["cost_trajectory"],
                         rep["termination"], rep["condition_warnings"])
    return report, _correction(graph, before)
