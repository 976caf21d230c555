"""Device-resident VI-BA problem: packed layout upload + thin wrappers over the C ABI.

``DeviceProblem`` turns the packed problem dict (``problem.pack_graph``) into
the device layout of include/vba.h:

* edges sorted (stably) by source keyframe, so each source's out-edges are a
  contiguous range the per-pixel kernels loop over;
* per-keyframe disparity segments and per-edge target/weight rows padded to a
  multiple of 4 pixels (16-byte aligned float4 loads of two pixels);
  padding pixels carry weight 0 and disparity 1 and never reach the caller;
* pixel coordinates implicit (regular grid, exact) when every keyframe and
  edge uses the same grid, else explicit per keyframe, else per edge;
* flow targets, weights, disparities in fp32; states, IMU factors, gravity fp64.

PyTorch provides device memory and the CUDA stream only.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L


def _require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2512_02293_b200 needs a CUDA device (sm_100a); there is no CPU fallback")


def _grid_params(X):
    """(ox, oy, sx, sy, W) if X (N,2) is exactly a row-major regular grid, else None."""
    N = len(X)
    if N == 0:
        return None
    ox, oy = float(X[0, 0]), float(X[0, 1])
    W = int(np.argmax(X[:, 1] != oy)) if np.any(X[:, 1] != oy) else N
    sx = float(X[1, 0] - X[0, 0]) if W > 1 else 1.0
    sy = float(X[W, 1] - oy) if W < N else 1.0
    n = np.arange(N)
    rec = np.stack([ox + sx * (n % W), oy + sy * (n // W)], 1)
    return (ox, oy, sx, sy, W) if np.array_equal(rec, X) else None


def detect_pixel_mode(P):
    K = len(P["kid"])
    doff, eoff = P["doff"], P["eoff"]
    for e in range(len(P["ei"])):
        i = P["ei"][e]
        a = P["epix"][eoff[e]:eoff[e + 1]]
        b = P["pix"][doff[i]:doff[i + 1]]
        if a.shape != b.shape or not np.array_equal(a, b):
            return L.PIX_EDGE, None
    gp = None
    for k in range(K):
        X = P["pix"][doff[k]:doff[k + 1]]
        if len(X) == 0:
            continue
        g = _grid_params(X)
        if g is None or (gp is not None and g != gp):
            return L.PIX_KF, None
        gp = g
    if gp is None:
        return L.PIX_KF, None
    return L.PIX_GRID, gp


def imu_records(P):
    F = len(P["fi"])
    R = np.zeros((F, L.IMU_REC))
    if F == 0:
        return R
    R[:, 0] = P["f_dt"]
    R[:, 1:5] = P["f_dR"]
    R[:, 5:8] = P["f_dp"]
    R[:, 8:11] = P["f_dv"]
    R[:, 11:20] = P["f_Jr"].reshape(F, 9)
    R[:, 20:38] = P["f_Jp"].reshape(F, 18)
    R[:, 38:56] = P["f_Jv"].reshape(F, 18)
    R[:, 56:137] = P["f_cov"][:, :9, :9].reshape(F, 81)
    R[:, 137:173] = P["f_cov"][:, 9:15, 9:15].reshape(F, 36)
    R[:, 173:179] = P["f_bhat"]
    return R


class HostLayout:
    """Padded, source-sorted host arrays (numpy) ready for upload."""

    def __init__(self, P, opts, edge_subset=None, imu_subset=None):
        K = len(P["kid"])
        self.K = K
        doff = np.asarray(P["doff"], np.int64)
        npix = (doff[1:] - doff[:-1]).astype(np.int64)
        npad = (npix + 3) // 4 * 4
        self.npix = npix.astype(np.int32)
        self.doff_pad = np.concatenate([[0], np.cumsum(npad)]).astype(np.int64)
        self.doff = doff
        ei_all = np.asarray(P["ei"], np.int64)
        eidx = np.arange(len(ei_all)) if edge_subset is None else np.asarray(edge_subset, np.int64)
        order = eidx[np.argsort(ei_all[eidx], kind="stable")]
        self.edge_order = order
        ei = ei_all[order]
        ej = np.asarray(P["ej"], np.int64)[order]
        E = len(order)
        self.E = E
        rows_pad = npad[ei] if E else np.zeros(0, np.int64)
        self.eoff_pad = (np.concatenate([[0], np.cumsum(rows_pad)])[:-1] if E else np.zeros(0)).astype(np.int64)
        n_rows_pad = int(rows_pad.sum()) if E else 0
        src = np.full(n_rows_pad, -1, np.int64)
        eoff = np.asarray(P["eoff"], np.int64)
        for k, e in enumerate(order):
            n = int(eoff[e + 1] - eoff[e])
            src[self.eoff_pad[k]:self.eoff_pad[k] + n] = np.arange(eoff[e], eoff[e] + n)
        valid = src >= 0
        self.tgt = np.zeros((n_rows_pad, 2), np.float32)
        self.w = np.zeros((n_rows_pad, 2), np.float32)
        # flow targets relative to the source pixel, u* - u (fp64 difference, then fp32):
        # the kernels predict the displacement, keeping fp32 error proportional to the flow
        self.tgt[valid] = P["tgt"][src[valid]] - P["epix"][src[valid]]
        self.w[valid] = P["w"][src[valid]]
        self.n_rows_pad = n_rows_pad
        n_disp_pad = int(self.doff_pad[-1])
        self.n_disp_pad = n_disp_pad
        dsrc = np.full(n_disp_pad, -1, np.int64)
        for k in range(K):
            dsrc[self.doff_pad[k]:self.doff_pad[k] + npix[k]] = np.arange(doff[k], doff[k + 1])
        self.dsrc = dsrc
        self.disp = np.ones(n_disp_pad, np.float32)
        self.disp[dsrc >= 0] = P["disp"][dsrc[dsrc >= 0]]
        self.mode, self.grid = detect_pixel_mode(P)
        if self.mode == L.PIX_KF:
            self.pix = np.zeros((n_disp_pad, 2), np.float32)
            self.pix[dsrc >= 0] = P["pix"][dsrc[dsrc >= 0]]
        elif self.mode == L.PIX_EDGE:
            self.pix = np.zeros((n_rows_pad, 2), np.float32)
            self.pix[valid] = P["epix"][src[valid]]
        else:
            self.pix = None
        self.ei = ei.astype(np.int32)
        self.ej = ej.astype(np.int32)
        fi = np.asarray(P["fi"], np.int64)
        fidx = np.arange(len(fi)) if imu_subset is None else np.asarray(imu_subset, np.int64)
        self.fi = fi[fidx].astype(np.int32)
        self.fj = np.asarray(P["fj"], np.int64)[fidx].astype(np.int32)
        self.imu = imu_records(P)[fidx] if len(fidx) else np.zeros((0, L.IMU_REC))
        self.F = len(fidx)
        self.state = np.concatenate([P["q"], P["p"], P["v"], P["bg"], P["ba"]], axis=1).astype(np.float64)
        self.ts = np.asarray(P["ts"], np.float64)
        self.grav = np.concatenate([P["grav_q"], [P["grav_G"]]]).astype(np.float64)
        frozen = set(int(k) for k in opts.get("frozen_keyframes", (0,)))
        self.frozen = np.array([int(k) in frozen for k in P["kid"]], np.int32)
        self.intr = np.asarray(P["intr"], np.float64)
        self.has_Tcb = bool(P.get("has_Tcb", False))
        self.Tcb = np.asarray(P["Tcb"], np.float64)


_TERM = {0: "max_iterations", 1: "converged", 2: "no_decrease_at_max_damping",
         3: "singular: singular reduced pose system"}


class DeviceProblem:
    """One VI-BA problem resident on the current CUDA device."""

    def __init__(self, P, opts: dict, layout: HostLayout | None = None, device=None, stream=None):
        _require_cuda()
        self.lib = L.load()
        self.opts = dict(opts)
        self.H = layout if layout is not None else HostLayout(P, self.opts)
        H = self.H
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        dev = self.device

        def t(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt, non_blocking=False)

        self.d_state = t(H.state, torch.float64)
        self.d_ts = t(H.ts, torch.float64)
        self.d_disp = t(H.disp, torch.float32)
        self.d_tgt = t(H.tgt.reshape(-1), torch.float32)
        self.d_w = t(H.w.reshape(-1), torch.float32)
        self.d_pix = t(H.pix.reshape(-1), torch.float32) if H.pix is not None else None
        self.d_imu = t(H.imu.reshape(-1), torch.float64)
        self.d_grav = t(H.grav, torch.float64)
        self._create()

    def _create(self):
        H = self.H
        self._host_keep = [np.ascontiguousarray(a) for a in (
            H.doff_pad, H.npix, H.ei, H.ej, H.eoff_pad, H.fi, H.fj, H.frozen)]
        hk = self._host_keep
        p = L.VbaProblem()
        p.n_kf, p.n_edges, p.n_imu = H.K, H.E, H.F
        p.pixel_mode = H.mode
        p.n_disp_pad, p.n_rows_pad = H.n_disp_pad, H.n_rows_pad
        if H.mode == L.PIX_GRID:
            ox, oy, sx, sy, W = H.grid
            p.grid_ox, p.grid_oy, p.grid_sx, p.grid_sy, p.grid_w = ox, oy, sx, sy, W
        p.has_Tcb = int(H.has_Tcb)
        p.fx, p.fy, p.cx, p.cy = (float(v) for v in H.intr)
        for k in range(7):
            p.Tcb[k] = float(H.Tcb[k])
        p.state = self.d_state.data_ptr()
        p.ts = self.d_ts.data_ptr()
        p.disp = self.d_disp.data_ptr()
        p.pix = self.d_pix.data_ptr() if self.d_pix is not None else None
        p.tgt = self.d_tgt.data_ptr()
        p.wts = self.d_w.data_ptr()
        p.imu = self.d_imu.data_ptr()
        p.grav = self.d_grav.data_ptr()
        p.h_doff, p.h_npix, p.h_edge_i, p.h_edge_j, p.h_eoff, p.h_imu_i, p.h_imu_j, p.h_frozen = (
            a.ctypes.data for a in hk)
        o = self.opts
        op = L.VbaOptions()
        op.max_iterations = int(o.get("max_iterations", 10))
        op.damping = float(o.get("damping", 1e-4))
        op.damping_up = float(o.get("damping_up", 10.0))
        op.damping_down = float(o.get("damping_down", 0.5))
        op.rel_decrease_tol = float(o.get("rel_decrease_tol", 1e-8))
        op.step_tol = float(o.get("step_tol", 1e-10))
        op.max_damping = float(o.get("max_damping", 1e8))
        op.optimize_gravity = int(bool(o.get("optimize_gravity", False)))
        op.optimize_velocity_bias = int(bool(o.get("optimize_velocity_bias", True)))
        op.use_schur = int(bool(o.get("use_schur", True)))
        op.ridge = float(o.get("ridge", 1e-10))
        self._p, self._o = p, op
        self.sdof = 15 if op.optimize_velocity_bias else 6
        self.npv = H.K * self.sdof + (2 if op.optimize_gravity else 0)
        self.n_disp = int(H.npix.sum())
        ctx = C.c_void_p()
        rc = self.lib.vba_create(C.byref(ctx), C.byref(p), C.byref(op), self._sptr())
        if rc == L.VBA_E_COV:
            raise ValueError("non-PSD preintegration covariance")
        L.check(rc)
        self.ctx = ctx

    def _sptr(self):
        return C.c_void_p(self.stream.cuda_stream)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.vba_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- stage wrappers -------------------------------------------------------
    def energy(self):
        t, v, i = C.c_double(), C.c_double(), C.c_double()
        L.check(self.lib.vba_energy(self.ctx, self._sptr(), C.byref(t), C.byref(v), C.byref(i)))
        return t.value, v.value, i.value

    def linearize(self):
        L.check(self.lib.vba_linearize(self.ctx, self._sptr()))

    def export_normal_eq(self, with_hpd=True, hpd_cols=None):
        """Reference-layout (H_pp, H_pd, H_dd, g_p, g_d) as numpy fp64 (solver.py:173-251).

        ``hpd_cols``: return only these disparity columns of H_pd (gathered on the device)."""
        dev = self.device
        npv, nd = self.npv, self.n_disp
        Hpp = torch.empty((npv, npv), dtype=torch.float64, device=dev)
        gp = torch.empty(npv, dtype=torch.float64, device=dev)
        Hpd = torch.empty((npv, max(nd, 1)), dtype=torch.float64, device=dev) if with_hpd else None
        Hdd = torch.empty(max(nd, 1), dtype=torch.float64, device=dev)
        gd = torch.empty(max(nd, 1), dtype=torch.float64, device=dev)
        L.check(self.lib.vba_export_normal_eq(self.ctx, self._sptr(), Hpp.data_ptr(), gp.data_ptr(),
                                              Hpd.data_ptr() if Hpd is not None else None,
                                              Hdd.data_ptr(), gd.data_ptr()))
        if Hpd is not None:
            Hpd = Hpd[:, :nd] if hpd_cols is None else Hpd[:, torch.as_tensor(hpd_cols, device=dev)]
        out = [Hpp.cpu().numpy(), Hpd.cpu().numpy() if Hpd is not None else None,
               Hdd[:nd].cpu().numpy(), gp.cpu().numpy(), gd[:nd].cpu().numpy()]
        return tuple(out)

    def export_reduced(self, lam):
        """Reduced system (H_red, g_red) at damping ``lam`` (solver.py:272-285), numpy fp64."""
        n = int(self.lib.vba_reduced_dim(self.ctx))
        Hr = torch.empty((max(n, 1), max(n, 1)), dtype=torch.float64, device=self.device)
        gr = torch.empty(max(n, 1), dtype=torch.float64, device=self.device)
        L.check(self.lib.vba_export_reduced(self.ctx, self._sptr(), float(lam), Hr.data_ptr(), gr.data_ptr()))
        return Hr[:n, :n].cpu().numpy(), gr[:n].cpu().numpy()

    def solve_step(self, lam, use_schur=True):
        """_solve_step (solver.py:265-308): returns (dx_full, dx_d) numpy fp64."""
        rc = self.lib.vba_solve_step(self.ctx, self._sptr(), float(lam), int(bool(use_schur)))
        if rc == L.VBA_E_NOT_SPD:
            raise RuntimeError("singular reduced pose system")
        L.check(rc)
        dx = torch.empty(self.npv, dtype=torch.float64, device=self.device)
        dxd = torch.empty(max(self.n_disp, 1), dtype=torch.float64, device=self.device)
        L.check(self.lib.vba_export_step(self.ctx, self._sptr(), dx.data_ptr(), dxd.data_ptr()))
        return dx.cpu().numpy(), dxd[:self.n_disp].cpu().numpy()

    def trial(self, lam, use_schur=True):
        r = L.VbaTrialResult()
        L.check(self.lib.vba_trial(self.ctx, self._sptr(), float(lam), int(bool(use_schur)), C.byref(r)))
        return r.status, r.new_cost, r.step_inf

    def accept(self):
        L.check(self.lib.vba_accept(self.ctx, self._sptr()))

    def solve(self):
        """Native LM loop (solver.py:344-411).  Returns a report dict."""
        cap = 4 * int(self._o.max_iterations) + 8
        traj = (C.c_double * cap)()
        rep = L.VbaReport()
        L.check(self.lib.vba_solve(self.ctx, self._sptr(), C.byref(rep), traj, cap))
        return dict(iterations=rep.iterations, initial_cost=rep.initial_cost, final_cost=rep.final_cost,
                    cost_trajectory=[traj[i] for i in range(min(rep.n_costs, cap))],
                    termination=_TERM[rep.termination],
                    condition_warnings=["singular reduced pose system"] * rep.n_warnings,
                    trials=rep.trials)

    def solve_windows(self, windows, outputs=None, copy_stream=None):
        """Solve a sequence of windows of this problem's topology end to end from host memory.

        ``windows``: dicts of (ideally pinned) host tensors in HostLayout order and dtype,
        keys ``state, disp, tgt, w, imu, grav``.  Window s+1's flow targets and weights
        (the bulk of the bytes) are uploaded on ``copy_stream`` into a second device set
        while window s is solved (``vba_bind_inputs`` swaps the sets); the small arrays are
        uploaded on the solve stream.  Each window's solved state and disparities are read
        back into ``outputs[s] = (state, disp)`` (pinned host tensors, allocated when not
        given) before the next window starts.  Returns the per-window reports."""
        if not windows:
            return []
        dev, st = self.device, self.stream
        cs = copy_stream if copy_stream is not None else torch.cuda.Stream(dev)
        if getattr(self, "_stage", None) is None:
            self._stage = (torch.empty_like(self.d_tgt), torch.empty_like(self.d_w))
        sets = ((self.d_tgt, self.d_w), self._stage)
        up = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        used = [False, False]

        def upload(s, b):
            with torch.cuda.stream(cs):
                if used[b]:
                    cs.wait_event(free[b])
                sets[b][0].copy_(windows[s]["tgt"].reshape(-1), non_blocking=True)
                sets[b][1].copy_(windows[s]["w"].reshape(-1), non_blocking=True)
                up[b].record(cs)

        if outputs is None:
            outputs = [(torch.empty(self.d_state.shape, dtype=torch.float64).pin_memory(),
                        torch.empty(self.d_disp.shape, dtype=torch.float32).pin_memory()) for _ in windows]
        cs.wait_stream(st)
        upload(0, 0)
        reps = []
        for s, win in enumerate(windows):
            b = s & 1
            if s + 1 < len(windows):
                upload(s + 1, b ^ 1)
            st.wait_event(up[b])
            with torch.cuda.stream(st):
                self.d_state.copy_(win["state"].reshape(self.d_state.shape), non_blocking=True)
                self.d_disp.copy_(win["disp"].reshape(self.d_disp.shape), non_blocking=True)
                self.d_imu.copy_(win["imu"].reshape(-1), non_blocking=True)
                self.d_grav.copy_(win["grav"].reshape(-1), non_blocking=True)
            rc = self.lib.vba_bind_inputs(self.ctx, self._sptr(), sets[b][0].data_ptr(), sets[b][1].data_ptr(), 1)
            if rc == L.VBA_E_COV:
                raise ValueError("non-PSD preintegration covariance")
            L.check(rc)
            self.load_state()
            reps.append(self.solve())
            L.check(self.lib.vba_download(self.ctx, self._sptr()))
            with torch.cuda.stream(st):
                outputs[s][0].copy_(self.d_state, non_blocking=True)
                outputs[s][1].copy_(self.d_disp, non_blocking=True)
            free[b].record(st)
            used[b] = True
        # leave the problem bound to its own arrays (window 0's set)
        st.wait_event(up[0])
        L.check(self.lib.vba_bind_inputs(self.ctx, self._sptr(), self.d_tgt.data_ptr(), self.d_w.data_ptr(), 0))
        return reps

    def download(self):
        """Current state as numpy: (q, p, v, bg, ba, disp[unpadded], grav_q)."""
        L.check(self.lib.vba_download(self.ctx, self._sptr()))
        self.stream.synchronize()
        s = self.d_state.cpu().numpy()
        d = self.d_disp.cpu().numpy().astype(np.float64)
        g = self.d_grav.cpu().numpy()
        disp = d[self.H.dsrc >= 0]
        return dict(q=s[:, 0:4], p=s[:, 4:7], v=s[:, 7:10], bg=s[:, 10:13], ba=s[:, 13:16], disp=disp,
                    grav_q=g[:4])

    def launch_count(self):
        return int(self.lib.vba_launch_count(self.ctx))

    def load_state(self):
        """Re-seed the solver state from the uploaded problem arrays."""
        L.check(self.lib.vba_load_state(self.ctx, self._sptr()))

    def set_profiling(self, on=True):
        L.check(self.lib.vba_set_profiling(self.ctx, int(bool(on))))

    def stage_times(self):
        out = (C.c_double * 7)()
        L.check(self.lib.vba_stage_times(self.ctx, out))
        return dict(zip(("linearize", "gram_fill", "assemble_chol", "backsub_retract", "energy", "k1_kernel",
                         "k1_launches"), list(out)))

    def solve_times(self):
        """Tensor-core reduced solve: factorisation / refinement ms, solves timed, n."""
        out = (C.c_double * 4)()
        L.check(self.lib.vba_solve_times(self.ctx, out))
        return dict(zip(("factor_ms", "refine_ms", "solves", "n"), list(out)))

    def stats(self):
        """[tensor-core solve enabled, fp64 fallbacks, tensor-core solves, refinement passes]."""
        out = (C.c_int64 * 4)()
        L.check(self.lib.vba_stats(self.ctx, out))
        return dict(zip(("tc_enabled", "fallbacks", "tc_solves", "refine_passes"), list(out)))

    def upload_inputs(self, H: "HostLayout" = None):
        """Re-upload the per-step inputs (host -> device copies of flow, weights,
        disparities, states, IMU records, gravity) from the host layout."""
        H = H or self.H
        for dst, src in ((self.d_state, H.state), (self.d_disp, H.disp), (self.d_tgt, H.tgt.reshape(-1)),
                         (self.d_w, H.w.reshape(-1)), (self.d_imu, H.imu.reshape(-1)), (self.d_grav, H.grav)):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src)), non_blocking=True)
