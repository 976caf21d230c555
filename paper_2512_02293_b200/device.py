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
* flow targets, weights in fp32; disparities as an fp64 master copy (the solver state,
  updated in fp64 like solver.py:336-338) plus its fp32 rounding (what the per-pixel
  kernels read); states, IMU factors, gravity fp64.

PyTorch provides device memory and the CUDA stream only.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib as L


def _require_cuda():
    if not L.cuda_available():
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


def _f64(a):
    return a if (type(a) is np.ndarray and a.dtype == np.float64) else np.asarray(a, dtype=np.float64)


class _PackedSource:
    """Layout source over a packed problem dict (``problem.pack_graph``; already validated)."""

    def __init__(self, P):
        self.P = P
        self.K = len(P["kid"])
        self.kid = np.asarray(P["kid"], np.int64)
        self.doff = np.asarray(P["doff"], np.int64)
        self.npix = (self.doff[1:] - self.doff[:-1]).astype(np.int64)
        self.ei = np.asarray(P["ei"], np.int64)
        self.ej = np.asarray(P["ej"], np.int64)
        self.eoff = np.asarray(P["eoff"], np.int64)
        self.state = np.concatenate([P["q"], P["p"], P["v"], P["bg"], P["ba"]], axis=1).astype(np.float64)
        self.ts = np.asarray(P["ts"], np.float64)
        self.grav = np.concatenate([P["grav_q"], [P["grav_G"]]]).astype(np.float64)
        self.intr = np.asarray(P["intr"], np.float64)
        self.has_Tcb = bool(P.get("has_Tcb", False))
        self.Tcb = np.asarray(P["Tcb"], np.float64)
        self.fi = np.asarray(P["fi"], np.int64)
        self.fj = np.asarray(P["fj"], np.int64)
        self._imu = None
        self.kpix = [P["pix"][self.doff[k]:self.doff[k + 1]] for k in range(self.K)]
        self.kdisp = [P["disp"][self.doff[k]:self.doff[k + 1]] for k in range(self.K)]

    def imu(self, idx):
        if self._imu is None:
            self._imu = imu_records(self.P)
        return self._imu[idx]

    def edge(self, e):
        r0, r1 = self.eoff[e], self.eoff[e + 1]
        P = self.P
        return P["epix"][r0:r1], P["tgt"][r0:r1], P["w"][r0:r1]


class _GraphSource:
    """Layout source read straight from a reference-style FrameGraph (duck-typed), with the
    validation of ``problem.pack_graph`` (residuals.py:181-185, 281-284)."""

    def __init__(self, graph):
        kfs = list(graph.keyframes)
        K = len(kfs)
        self.K = K
        self.kid = np.array([kf.kid for kf in kfs], dtype=np.int64)
        index = {int(k): n for n, k in enumerate(self.kid)}
        st = np.empty((K, 16))
        ts = np.empty(K)
        self.kpix, self.kdisp = [], []
        for n, kf in enumerate(kfs):
            s = kf.state
            st[n, 0:4] = s.pose.rotation.q
            st[n, 4:7] = s.pose.translation
            st[n, 7:10] = s.velocity
            st[n, 10:13] = s.bias.gyro_bias
            st[n, 13:16] = s.bias.accel_bias
            ts[n] = s.timestamp
            d = _f64(kf.disparities).reshape(-1)
            if len(d) and d.min() <= 0.0:
                raise ValueError("disparities must be strictly positive")
            self.kdisp.append(d)
            self.kpix.append(_f64(kf.pixels).reshape(-1, 2))
        self.state, self.ts = st, ts
        self.npix = np.array([len(d) for d in self.kdisp], dtype=np.int64)
        self.doff = np.concatenate([[0], np.cumsum(self.npix)]).astype(np.int64)
        edges = list(graph.vision_edges)
        self.edges = edges
        self.ei = np.array([index[e.i] for e in edges], dtype=np.int64)
        self.ej = np.array([index[e.j] for e in edges], dtype=np.int64)
        rows = np.array([len(e.pixels) for e in edges], dtype=np.int64)
        if len(edges) and np.any(rows != self.npix[self.ei]):
            raise ValueError("disparity length must match edge pixel list")
        self.eoff = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
        ies = list(graph.inertial_edges)
        F = len(ies)
        self.fi = np.array([index[i] for i, _, _ in ies], dtype=np.int64)
        self.fj = np.array([index[j] for _, j, _ in ies], dtype=np.int64)
        R = np.zeros((F, L.IMU_REC))
        for f, (_, _, d) in enumerate(ies):
            r = R[f]
            r[0] = d.dt_total
            r[1:5] = d.delta_R.q
            r[5:8] = d.delta_p
            r[8:11] = d.delta_v
            r[11:20] = np.asarray(d.J_rot, float).reshape(9)
            r[20:38] = np.asarray(d.J_pos, float).reshape(18)
            r[38:56] = np.asarray(d.J_vel, float).reshape(18)
            cov = np.asarray(d.covariance, float).reshape(15, 15)
            r[56:137] = cov[:9, :9].reshape(81)
            r[137:173] = cov[9:15, 9:15].reshape(36)
            r[173:176] = d.bias_lin_point.gyro_bias
            r[176:179] = d.bias_lin_point.accel_bias
        if F:
            dts = ts[self.fj] - ts[self.fi]
            bad = np.nonzero(np.abs(dts - R[:, 0]) > 1e-6)[0]
            if len(bad):
                f = int(bad[0])
                raise ValueError(f"delta spans {R[f, 0]:.6f}s but states are {dts[f]:.6f}s apart")
        self._imu = R
        g = graph.gravity
        self.grav = np.concatenate([np.asarray(g.R_wg.q, float), [float(g.magnitude)]])
        k = graph.intrinsics
        self.intr = np.array([k.fx, k.fy, k.cx, k.cy], dtype=float)
        T = getattr(graph, "T_cb", None)
        self.has_Tcb = T is not None
        self.Tcb = (np.concatenate([np.asarray(T.rotation.q, float), np.asarray(T.translation, float)])
                    if T is not None else np.array([1.0, 0, 0, 0, 0, 0, 0]))

    def imu(self, idx):
        return self._imu[idx]

    def edge(self, e):
        x = self.edges[e]
        return _f64(x.pixels), _f64(x.targets), _f64(x.weights)


def _same_buffer(a, b):
    """a and b view the same memory with the same layout (e.g. an edge sharing its source
    keyframe's pixel array), so their contents are equal without reading them."""
    if a is b:
        return True
    ia, ib = a.__array_interface__, b.__array_interface__
    return ia["data"][0] == ib["data"][0] and a.shape == b.shape and a.strides == b.strides and a.dtype == b.dtype


def _host_buffer(shape, dtype, pinned):
    """Zero-free host buffer; page-locked (torch's caching host allocator) when ``pinned``."""
    if pinned:
        tdt = {np.float32: torch.float32, np.float64: torch.float64}[dtype]
        t = torch.empty(shape, dtype=tdt, pin_memory=True)
        return t.numpy(), t
    return np.empty(shape, dtype), None


_POOL = None


def _pack_threads(total_rows):
    n = int(os.environ.get("VBA_PACK_THREADS", "0")) or min(32, os.cpu_count() or 1)
    return 1 if total_rows < (1 << 16) else n


def _pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1), thread_name_prefix="vba-pack")
    return _POOL


class HostLayout:
    """Padded, source-sorted host arrays (numpy) ready for upload.

    Built from a packed problem dict (``HostLayout(P, opts)``) or straight from a
    FrameGraph (``HostLayout.from_graph``); both run the same fill, so the arrays are
    bitwise identical.  Flow targets are stored relative to the source pixel,
    u* - u, computed in fp64 and rounded once to fp32 (the kernels predict the
    displacement, which keeps fp32 error proportional to the flow).  The per-edge
    fill runs on a thread pool (numpy releases the GIL in its loops) into page-locked
    buffers when ``pinned``, so the upload is one asynchronous DMA per array.
    """

    def __init__(self, P, opts, edge_subset=None, imu_subset=None, pinned=False, _src=None):
        self._build(_src if _src is not None else _PackedSource(P), opts, edge_subset, imu_subset, pinned)

    @classmethod
    def from_graph(cls, graph, opts, pinned=None):
        if pinned is None:
            pinned = L.cuda_available()
        return cls(None, opts, pinned=pinned, _src=_GraphSource(graph))

    def _build(self, S, opts, edge_subset, imu_subset, pinned):
        K = S.K
        self.K = K
        npix = S.npix
        npad = (npix + 3) // 4 * 4
        self.npix = npix.astype(np.int32)
        self.doff = S.doff
        self.doff_pad = np.concatenate([[0], np.cumsum(npad)]).astype(np.int64)
        eidx = np.arange(len(S.ei)) if edge_subset is None else np.asarray(edge_subset, np.int64)
        order = eidx[np.argsort(S.ei[eidx], kind="stable")]
        self.edge_order = order
        ei, ej = S.ei[order], S.ej[order]
        E = len(order)
        self.E = E
        rows = (S.eoff[order + 1] - S.eoff[order]) if E else np.zeros(0, np.int64)
        rows_pad = npad[ei] if E else np.zeros(0, np.int64)
        self.eoff_pad = (np.concatenate([[0], np.cumsum(rows_pad)])[:-1] if E else np.zeros(0)).astype(np.int64)
        n_rows_pad = int(rows_pad.sum()) if E else 0
        self.n_rows_pad = n_rows_pad
        self.tgt, self._tgt_t = _host_buffer((n_rows_pad, 2), np.float32, pinned)
        self.w, self._w_t = _host_buffer((n_rows_pad, 2), np.float32, pinned)

        kpix = S.kpix
        # weight signs: checked while packing by the native packer (graph sources: the weights
        # are read there anyway) and for host-only layouts; pinned packed-dict layouts are
        # checked on the device after the upload (DeviceProblem), which reads the fp32 copy at
        # HBM speed instead of the fp64 source
        self.weights_checked = not pinned or isinstance(S, _GraphSource)
        neg = self._fill_edges(S, order, ei, rows, rows_pad, kpix, check_neg=self.weights_checked)
        if neg:
            raise ValueError("weights must be non-negative")

        n_disp_pad = int(self.doff_pad[-1])
        self.n_disp_pad = n_disp_pad
        n_real = int(S.doff[-1])
        kk = np.repeat(np.arange(K), npix)
        pos = np.arange(n_real) - S.doff[kk] + self.doff_pad[kk]      # padded slot of every real pixel
        dsrc = np.full(n_disp_pad, -1, np.int64)
        dsrc[pos] = np.arange(n_real)
        self.dsrc = dsrc
        self.disp64, self._disp_t = _host_buffer(n_disp_pad, np.float64, pinned)
        self.disp64.fill(1.0)
        for k in range(K):
            if npix[k]:
                self.disp64[self.doff_pad[k]:self.doff_pad[k] + npix[k]] = S.kdisp[k]
        self.disp = self.disp64.astype(np.float32)
        self.mode, self.grid = self._pixel_mode(kpix, self._edge_mismatch)
        if self.mode == L.PIX_KF:
            self.pix = np.zeros((n_disp_pad, 2), np.float32)
            for k in range(K):
                self.pix[self.doff_pad[k]:self.doff_pad[k] + npix[k]] = kpix[k]
        elif self.mode == L.PIX_EDGE:
            self.pix = np.zeros((n_rows_pad, 2), np.float32)
            for k, e in enumerate(order):
                self.pix[self.eoff_pad[k]:self.eoff_pad[k] + rows[k]] = S.edge(e)[0]
        else:
            self.pix = None
        self.ei = ei.astype(np.int32)
        self.ej = ej.astype(np.int32)
        fidx = np.arange(len(S.fi)) if imu_subset is None else np.asarray(imu_subset, np.int64)
        self.fi = S.fi[fidx].astype(np.int32)
        self.fj = S.fj[fidx].astype(np.int32)
        self.imu = S.imu(fidx) if len(fidx) else np.zeros((0, L.IMU_REC))
        self.F = len(fidx)
        self.state = S.state
        self.ts = S.ts
        self.grav = S.grav
        frozen = set(int(k) for k in opts.get("frozen_keyframes", (0,)))
        self.frozen = np.array([int(k) in frozen for k in S.kid], np.int32)
        self.intr = S.intr
        self.has_Tcb = S.has_Tcb
        self.Tcb = S.Tcb

    def _fill_edges(self, S, order, ei, rows, rows_pad, kpix, check_neg=True):
        """flow (u* - u, fp64 difference rounded to fp32) and weights of every edge into the
        padded rows; records whether any edge's pixels differ from its source keyframe's.

        Graph sources go through the native packer (csrc/vba_pack.cpp: buffer protocol,
        GIL released, one thread per row range); packed dicts through numpy slices."""
        T, W, eoff_pad = self.tgt, self.w, self.eoff_pad
        if isinstance(S, _GraphSource):
            from . import _vbapack
            mism, neg = _vbapack.pack_edges(
                S.edges, np.ascontiguousarray(order, np.int64), np.ascontiguousarray(ei, np.int64),
                np.ascontiguousarray(rows, np.int64), np.ascontiguousarray(eoff_pad, np.int64),
                np.ascontiguousarray(rows_pad, np.int64), kpix, T.reshape(-1), W.reshape(-1),
                _pack_threads(int(rows.sum()) if len(rows) else 0), int(check_neg))
            self._edge_mismatch = bool(mism)
            return bool(neg)

        def run(k0, k1):
            mism = neg = False
            for k in range(k0, k1):
                pix, tgt, w = S.edge(order[k])
                r0 = eoff_pad[k]
                r1 = r0 + rows[k]
                rp = r0 + rows_pad[k]
                np.subtract(tgt, pix, out=T[r0:r1], casting="unsafe")
                np.copyto(W[r0:r1], w, casting="unsafe")
                if rp > r1:
                    T[r1:rp] = 0.0
                    W[r1:rp] = 0.0
                if check_neg and rows[k] and w.min() < 0.0:
                    neg = True
                if not mism:
                    kp = kpix[ei[k]]
                    mism = not (_same_buffer(pix, kp) or (pix.shape == kp.shape and np.array_equal(pix, kp)))
            return mism, neg

        E = len(order)
        total = int(rows.sum()) if E else 0
        if total < (1 << 18) or E < 16:
            res = [run(0, E)]
        else:
            nch = min(8 * min(16, os.cpu_count() or 1), E)
            cuts = np.linspace(0, E, nch + 1).astype(int)
            res = list(_pool().map(lambda ab: run(*ab), zip(cuts[:-1], cuts[1:])))
        self._edge_mismatch = any(m for m, _ in res)
        return any(n for _, n in res)

    @staticmethod
    def _pixel_mode(kpix, edge_mismatch):
        """VBA_PIX_GRID when every keyframe uses the same exact regular grid and every edge
        the pixels of its source keyframe; VBA_PIX_KF / VBA_PIX_EDGE otherwise."""
        if edge_mismatch:
            return L.PIX_EDGE, None
        gp = None
        first = None
        seen = {}
        for X in kpix:
            if len(X) == 0:
                continue
            g = seen.get(id(X))
            if g is None:
                if first is not None and X.shape == first[0].shape and np.array_equal(X, first[0]):
                    g = first[1]
                else:
                    g = _grid_params(X) or False
                seen[id(X)] = g
                if first is None:
                    first = (X, g)
            if g is False or (gp is not None and g != gp):
                return L.PIX_KF, None
            gp = g
        if gp is None:
            return L.PIX_KF, None
        return L.PIX_GRID, gp

    def pinned_tensors(self):
        """(tgt, w, disp64) page-locked torch views, or None when built unpinned."""
        if self._tgt_t is None:
            return None
        return self._tgt_t, self._w_t, self._disp_t


_TERM = {0: "max_iterations", 1: "converged", 2: "no_decrease_at_max_damping"}


class DeviceProblem:
    """One VI-BA problem resident on the current CUDA device."""

    def __init__(self, P, opts: dict, layout: HostLayout | None = None, device=None, stream=None, shard=None):
        """``shard = (rank, world, kbounds)``: an edge-sharded rank of a multi-GPU solve
        (paper_2512_02293_b200.distributed); the layout is the whole problem."""
        _require_cuda()
        self.lib = L.load()
        self.opts = dict(opts)
        self.shard = shard
        self.H = layout if layout is not None else HostLayout(P, self.opts)
        H = self.H
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        dev = self.device

        with torch.cuda.stream(self.stream):
            self.d_state = torch.empty((H.K, 16), dtype=torch.float64, device=dev)
            self.d_ts = torch.empty(H.K, dtype=torch.float64, device=dev)
            self.d_disp = torch.empty(H.n_disp_pad, dtype=torch.float32, device=dev)
            self.d_disp64 = torch.empty(H.n_disp_pad, dtype=torch.float64, device=dev)
            self.d_tgt = torch.empty(2 * H.n_rows_pad, dtype=torch.float32, device=dev)
            self.d_w = torch.empty(2 * H.n_rows_pad, dtype=torch.float32, device=dev)
            self.d_pix = (torch.empty(H.pix.size, dtype=torch.float32, device=dev) if H.pix is not None else None)
            self.d_imu = torch.empty(H.F * L.IMU_REC, dtype=torch.float64, device=dev)
            self.d_grav = torch.empty(5, dtype=torch.float64, device=dev)
        self._upload(H)
        self._create()

    def _upload(self, H):
        """Host layout -> this problem's device arrays, on the solve stream.  The bulk arrays
        (flow, weights, disparities) go as asynchronous DMAs from page-locked buffers when the
        layout was built pinned; weight signs are then checked on the device (ValueError, as
        residuals.py:112-113)."""
        pin = H.pinned_tensors() if hasattr(H, "pinned_tensors") else None
        with torch.cuda.stream(self.stream):
            def put(dst, a, pinned=None):
                if dst is None or dst.numel() == 0:
                    return
                if pinned is not None:
                    dst.copy_(pinned.reshape(-1), non_blocking=True)
                elif isinstance(a, torch.Tensor):   # device-resident source (window.DeviceWindow)
                    dst.copy_(a.reshape(-1), non_blocking=True)
                else:   # small host arrays: through page-locked staging (torch's caching host allocator), async
                    src = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(dst.dtype)
                    dst.copy_(src.pin_memory() if pin else src, non_blocking=pin is not None)
            put(self.d_state.view(-1), H.state)
            put(self.d_ts, H.ts)
            put(self.d_disp64, H.disp64, pin[2] if pin else None)   # the fp32 copy is derived natively
            put(self.d_tgt, H.tgt, pin[0] if pin else None)
            put(self.d_w, H.w, pin[1] if pin else None)
            put(self.d_pix, H.pix)
            put(self.d_imu, H.imu)
            put(self.d_grav, H.grav)
            if not H.weights_checked and self.d_w.numel() and bool((self.d_w < 0).any()):
                raise ValueError("weights must be non-negative")

    def rebind(self, H):
        """Solve another window of the same topology in this context (no re-planning):
        upload its arrays, re-derive the IMU whitening factors, reset the LM state."""
        self.H = H
        self._upload(H)
        rc = self.lib.vba_bind_inputs(self.ctx, self._sptr(), self.d_tgt.data_ptr(), self.d_w.data_ptr(), 1)
        if rc == L.VBA_E_COV:
            raise ValueError("non-PSD preintegration covariance")
        L.check(rc)
        self.load_state()

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
        p.disp64 = self.d_disp64.data_ptr()
        p.pix = self.d_pix.data_ptr() if self.d_pix is not None else None
        p.tgt = self.d_tgt.data_ptr()
        p.wts = self.d_w.data_ptr()
        p.imu = self.d_imu.data_ptr()
        p.grav = self.d_grav.data_ptr()
        p.h_doff, p.h_npix, p.h_edge_i, p.h_edge_j, p.h_eoff, p.h_imu_i, p.h_imu_j, p.h_frozen = (
            a.ctypes.data for a in hk)
        if self.shard is not None and self.shard[1] > 1:
            rank, world, kb = self.shard
            self._kb = np.ascontiguousarray(kb, np.int32)
            p.shard_world, p.shard_rank, p.h_shard_kbounds = int(world), int(rank), self._kb.ctypes.data
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
            dense = not use_schur and self.n_disp > 0
            raise RuntimeError("singular full system" if dense else "singular reduced pose system")
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

    def _singular_msg(self):
        """The reference's RuntimeError text for a singular step (solver.py:287-289, 300-303):
        the dense path is taken when use_schur is off and there are disparities."""
        dense = not bool(self.opts.get("use_schur", True)) and self.n_disp > 0
        return "singular full system" if dense else "singular reduced pose system"

    def _term(self, code):
        return _TERM[code] if code in _TERM else "singular: " + self._singular_msg()

    def solve(self):
        """Native LM loop (solver.py:344-411).  Returns a report dict."""
        cap = 4 * int(self._o.max_iterations) + 8
        traj = (C.c_double * cap)()
        rep = L.VbaReport()
        L.check(self.lib.vba_solve(self.ctx, self._sptr(), C.byref(rep), traj, cap))
        return dict(iterations=rep.iterations, initial_cost=rep.initial_cost, final_cost=rep.final_cost,
                    cost_trajectory=[traj[i] for i in range(min(rep.n_costs, cap))],
                    termination=self._term(rep.termination),
                    condition_warnings=[self._singular_msg()] * rep.n_warnings,
                    trials=rep.trials)

    def solve_windows(self, windows, outputs=None, copy_stream=None):
        """Solve a sequence of windows of this problem's topology end to end from host memory.

        ``windows``: dicts of (ideally pinned) host tensors in HostLayout order and dtype,
        keys ``state, disp64`` (fp64 disparities; or ``disp``, fp32), ``tgt, w, imu, grav``.  Keep the
        solve stream free of torch kernels in the loop: an fp32 ``disp`` needs a widening kernel,
        which on the legacy default stream serialises the copy stream's uploads with the solve
        (measured: 23.2 vs 14.8 ms per config-4 window).  Window s+1's flow targets and weights
        (the bulk of the bytes) are uploaded on ``copy_stream`` into a second device set
        while window s is solved (``vba_bind_inputs`` swaps the sets); the small arrays ride
        the same copy stream into staging buffers and are moved into place by device copies
        on the solve stream.  Each window's solved state and disparities are read
        back into ``outputs[s] = (state, disp)`` (pinned host tensors, allocated when not
        given) before the next window starts.  Returns the per-window reports."""
        if not windows:
            return []
        dev, st = self.device, self.stream
        cs = copy_stream if copy_stream is not None else torch.cuda.Stream(dev)
        if getattr(self, "_stage", None) is None:
            self._stage = (torch.empty_like(self.d_tgt), torch.empty_like(self.d_w))
        sets = ((self.d_tgt, self.d_w), self._stage)
        # the small per-window arrays travel on the copy stream too, into a device staging set
        # per buffer, and are moved into place by device copies on the solve stream: copies
        # from two streams share the host->device engine in no fixed order, so a small copy on
        # the solve stream could wait behind a whole 600 MB bulk upload of the next window
        small = ("state", "disp64", "imu", "grav")
        dst = {"state": self.d_state, "disp64": self.d_disp64, "imu": self.d_imu, "grav": self.d_grav}
        if getattr(self, "_stage_small", None) is None:
            self._stage_small = [{k: torch.empty(dst[k].numel(), dtype=dst[k].dtype, device=dev) for k in small}
                                 for _ in range(2)]
        up = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        used = [False, False]

        def upload(s, b):
            with torch.cuda.stream(cs):
                if used[b]:
                    cs.wait_event(free[b])
                win = windows[s]
                for k in small:
                    if k == "disp64" and k not in win:
                        continue
                    self._stage_small[b][k].copy_(win[k].reshape(-1), non_blocking=True)
                sets[b][0].copy_(win["tgt"].reshape(-1), non_blocking=True)
                sets[b][1].copy_(win["w"].reshape(-1), non_blocking=True)
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
            with torch.cuda.stream(st):   # device-to-device (kernels: no copy engine involved)
                for k in small:
                    if k == "disp64" and k not in win:
                        continue
                    dst[k].view(-1).copy_(self._stage_small[b][k])
                if "disp64" not in win:   # fp32 window disparities seed the fp64 master
                    self.d_disp.copy_(win["disp"].reshape(self.d_disp.shape), non_blocking=True)
                    self.d_disp64.copy_(self.d_disp)
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
        d = self.d_disp64.cpu().numpy()
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
        d = dict(zip(("tc_enabled", "fallbacks", "tc_solves", "refine_passes"), list(out)))
        d["gram_tc"] = int(self.lib.vba_gram_kind(self.ctx))
        return d

    def upload_inputs(self, H: "HostLayout" = None):
        """Re-upload the per-step inputs (host -> device copies of flow, weights,
        disparities, states, IMU records, gravity) from the host layout."""
        H = H or self.H
        for dst, src in ((self.d_state, H.state), (self.d_disp, H.disp), (self.d_disp64, H.disp64),
                         (self.d_tgt, H.tgt.reshape(-1)),
                         (self.d_w, H.w.reshape(-1)), (self.d_imu, H.imu.reshape(-1)), (self.d_grav, H.grav)):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src)), non_blocking=True)
