"""Device-resident tracking window.

The reference's tracker (/root/reference/pkg/src/vislam/frontend.py) rebuilds a
``FrameGraph`` of host arrays at every keyframe -- ``add_keyframe`` (:341-432) wires the
new keyframe's correspondence edges to its window neighbours, ``_tracking_solve``
(:435-450) runs ``solve_vi_ba`` on the window, ``_evict`` (:453-482) drops the oldest
keyframe with its edges and inertial factor -- so every solve re-packs and re-uploads the
whole window.  ``DeviceWindow`` keeps the window on the GPU instead:

* a keyframe's disparities (fp64 master copy) and an edge's flow targets / weights (fp32,
  the layout the kernels stream) are uploaded ONCE, when they are inserted;
* a solve gathers the window device-to-device into the solver's packed layout and reuses
  the solver context of the window's topology (the steady state of a tracker has one: the
  same covisibility pattern keyframe after keyframe), so no planning and no bulk
  host->device traffic happens per keyframe;
* the solved disparities are scattered back to the keyframes on the device; only the
  keyframe states ([K,16] fp64) come back to the host;
* eviction frees the oldest keyframe's buffers.

``from_tracker_dict`` replays a window serialised by the reference's
``TrackerState.to_dict`` (frontend.py:209-294, the JSON checkpoint format) into the device
window, and ``graph()`` returns the window as host objects.  A window solve is bitwise the
drop-in ``solver.solve_vi_ba`` on the same graph (same packed layout, same kernels).
"""

from __future__ import annotations

import ctypes as C
import hashlib
from collections import OrderedDict

import numpy as np
import torch

from . import _lib as L
from .device import DeviceProblem, _grid_params
from .types import SolveOptions, SolveReport


class _Kf:
    __slots__ = ("kid", "state", "ts", "pixels", "disp", "n", "grid")

    def __init__(self, kid, state16, ts, pixels, disp):
        self.kid, self.state, self.ts, self.pixels, self.disp = kid, state16, ts, pixels, disp
        self.n = len(pixels)
        self.grid = _grid_params(pixels) if self.n else None   # detected once, at insertion


class _Edge:
    __slots__ = ("i", "j", "flow", "w", "pixels")

    def __init__(self, i, j, flow, w, pixels):
        self.i, self.j, self.flow, self.w, self.pixels = i, j, flow, w, pixels


def _state16(st):
    return np.concatenate([np.asarray(st.pose.rotation.q, float), np.asarray(st.pose.translation, float),
                           np.asarray(st.velocity, float), np.asarray(st.bias.gyro_bias, float),
                           np.asarray(st.bias.accel_bias, float)])


def _imu_record(d):
    r = np.zeros(L.IMU_REC)
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
    return r


class _Staging:
    """Page-locked host staging for the window's uploads: insertions copy into it and
    enqueue asynchronous host->device copies on the current stream (no synchronising
    pageable copy per array); the buffer is recycled once the stream has drained them."""

    def __init__(self, device, nbytes=1 << 22):
        self.device = device
        self.buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        self.off = 0
        self.ev = None

    def put(self, a: np.ndarray, dtype) -> torch.Tensor:
        a = np.ascontiguousarray(a)
        n = a.nbytes
        if n == 0:
            return torch.empty(0, dtype=dtype, device=self.device)
        if self.off + n > self.buf.numel():
            self.recycle(wait=True)
            if n > self.buf.numel():
                self.buf = torch.empty(max(n, 2 * self.buf.numel()), dtype=torch.uint8, pin_memory=True)
        if self.off == 0 and self.ev is not None:   # earlier copies out of this buffer must be done
            self.ev.synchronize()
            self.ev = None
        o = (self.off + 255) // 256 * 256
        host = self.buf[o:o + n]
        host.numpy()[:] = a.view(np.uint8).reshape(-1)
        dev = torch.empty(n // np.dtype(a.dtype).itemsize, dtype=dtype, device=self.device)
        dev.view(torch.uint8).copy_(host, non_blocking=True)
        self.off = o + n
        return dev

    def recycle(self, wait=False):
        """Start over at the head of the buffer (after the copies queued so far)."""
        if self.off:
            self.ev = torch.cuda.Event()
            self.ev.record(torch.cuda.current_stream(self.device))
            if wait:
                self.ev.synchronize()
                self.ev = None
        self.off = 0


def _segments(segs, device, stage: "_Staging"):
    """One vba_copy_segments launch for a list of (src, dst, bytes) device copies."""
    if not segs:
        return
    tab = np.array(segs, dtype=np.int64).reshape(-1, 3)
    d = stage.put(tab, torch.int64)
    L.check(L.load().vba_copy_segments(C.c_void_p(d.data_ptr()), len(segs),
                                       C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))


class _WinLayout:
    """The attributes DeviceProblem reads from a HostLayout, with the bulk arrays on the device."""

    weights_checked = False

    def pinned_tensors(self):
        return None


class DeviceWindow:
    """A sliding VI-BA window resident on one GPU (frontend.py:341-482 semantics)."""

    def __init__(self, intrinsics, gravity=None, T_cb=None, window_size=12, device=None, cache_size=4):
        if not L.cuda_available():
            raise RuntimeError("paper_2512_02293_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        k = intrinsics
        self.intrinsics = intrinsics
        self.intr = np.array([k.fx, k.fy, k.cx, k.cy], dtype=float)
        if gravity is None:
            self.grav = np.array([1.0, 0.0, 0.0, 0.0, 9.81])
        else:
            self.grav = np.concatenate([np.asarray(gravity.R_wg.q, float), [float(gravity.magnitude)]])
        self.gravity_obj = gravity
        self.T_cb = T_cb
        self.Tcb = (np.concatenate([np.asarray(T_cb.rotation.q, float), np.asarray(T_cb.translation, float)])
                    if T_cb is not None else np.array([1.0, 0, 0, 0, 0, 0, 0]))
        self.window_size = window_size
        self.kfs: "OrderedDict[int, _Kf]" = OrderedDict()
        self.edges: list = []
        self.imu: "OrderedDict[tuple, np.ndarray]" = OrderedDict()
        self._cache: "OrderedDict[tuple, DeviceProblem]" = OrderedDict()
        self.cache_size = cache_size
        self.h2d_bytes = 0          # bulk bytes uploaded by insertions (instrumentation)
        self._stage = _Staging(self.device)
        self.solves = 0
        self.replans = 0

    # ---- window edits (frontend.py:341-432, 453-482) --------------------------------
    def add_keyframe(self, kid, state, pixels, disparities):
        pixels = np.asarray(pixels, float).reshape(-1, 2)
        d = np.asarray(disparities, float).reshape(-1)
        if len(d) != len(pixels):
            raise ValueError("one disparity per tracked pixel")
        if len(d) and d.min() <= 0.0:
            raise ValueError("disparities must be positive")
        if kid in self.kfs:
            raise ValueError(f"keyframe {kid} is already in the window")
        t = self._stage.put(d, torch.float64)
        self.h2d_bytes += d.nbytes
        self.kfs[kid] = _Kf(kid, _state16(state), float(state.timestamp), pixels, t)

    def add_vision_edge(self, i, j, pixels, targets, weights):
        if i not in self.kfs or j not in self.kfs:
            raise ValueError(f"vision edge ({i},{j}) references unknown keyframe")
        pixels = np.asarray(pixels, float).reshape(-1, 2)
        targets = np.asarray(targets, float).reshape(-1, 2)
        weights = np.asarray(weights, float).reshape(-1, 2)
        n = len(pixels)
        if len(targets) != n or len(weights) != n:
            raise ValueError("pixels, targets and weights must have equal length")
        if n != self.kfs[i].n:
            raise ValueError("disparity length must match edge pixel list")
        if np.any(weights < 0.0):
            raise ValueError("weights must be non-negative")
        flow = (targets - pixels).astype(np.float32)   # u* - u: fp64 difference, one rounding
        w = weights.astype(np.float32)
        same = np.array_equal(pixels, self.kfs[i].pixels)
        e = _Edge(i, j, self._stage.put(flow.reshape(-1), torch.float32),
                  self._stage.put(w.reshape(-1), torch.float32), None if same else pixels)
        self.h2d_bytes += flow.nbytes + w.nbytes
        self.edges.append(e)

    def add_inertial_edge(self, i, j, delta):
        self.imu[(i, j)] = _imu_record(delta)

    def evict(self, kid=None):
        """Drop keyframe ``kid`` (default: the oldest) with its vision edges and the inertial
        factors it starts (frontend.py:470-477)."""
        if kid is None:
            kid = next(iter(self.kfs))
        self.kfs.pop(kid)
        self.edges = [e for e in self.edges if e.i != kid and e.j != kid]
        for key in [k for k in self.imu if k[0] == kid]:
            self.imu.pop(key)

    def evict_to_size(self, pinned=()):
        """frontend._evict's loop: the oldest keyframe leaves while the window is too large,
        unless it is pinned."""
        while len(self.kfs) > self.window_size and next(iter(self.kfs)) not in pinned:
            self.evict()

    # ---- solve (frontend.py:435-450 -> solver.py:344-411) ------------------------------
    def _layout(self, opts, use_inertial=True):
        kids = list(self.kfs)
        index = {k: n for n, k in enumerate(kids)}
        K = len(kids)
        Ly = _WinLayout()
        Ly.K = K
        npix = np.array([self.kfs[k].n for k in kids], dtype=np.int64)
        npad = (npix + 3) // 4 * 4
        Ly.npix = npix.astype(np.int32)
        Ly.doff_pad = np.concatenate([[0], np.cumsum(npad)]).astype(np.int64)
        Ly.n_disp_pad = int(Ly.doff_pad[-1])
        src = np.array([index[e.i] for e in self.edges], dtype=np.int64)
        order = np.argsort(src, kind="stable")
        Ly.order = order
        Ly.ei = src[order].astype(np.int32)
        Ly.ej = np.array([index[self.edges[q].j] for q in order], dtype=np.int32)
        Ly.E = len(order)
        rows_pad = npad[Ly.ei] if Ly.E else np.zeros(0, np.int64)
        Ly.eoff_pad = (np.concatenate([[0], np.cumsum(rows_pad)])[:-1] if Ly.E else np.zeros(0)).astype(np.int64)
        Ly.n_rows_pad = int(rows_pad.sum()) if Ly.E else 0
        imu = ([(index[i], index[j], r) for (i, j), r in self.imu.items() if i in index and j in index]
               if use_inertial else [])
        Ly.F = len(imu)
        Ly.fi = np.array([a for a, _, _ in imu], dtype=np.int32)
        Ly.fj = np.array([b for _, b, _ in imu], dtype=np.int32)
        Ly.imu = np.array([r for _, _, r in imu]).reshape(Ly.F, L.IMU_REC)
        if Ly.F:
            dts = np.array([self.kfs[kids[b]].ts - self.kfs[kids[a]].ts for a, b, _ in imu])
            bad = np.nonzero(np.abs(dts - Ly.imu[:, 0]) > 1e-6)[0]
            if len(bad):
                raise ValueError(f"delta spans {Ly.imu[bad[0], 0]:.6f}s but states are {dts[bad[0]]:.6f}s apart")
        Ly.state = np.array([self.kfs[k].state for k in kids]).reshape(K, 16)
        Ly.ts = np.array([self.kfs[k].ts for k in kids])
        Ly.grav = self.grav.copy()
        frozen = set(int(k) for k in opts.get("frozen_keyframes", (kids[0],)))
        Ly.frozen = np.array([int(k) in frozen for k in kids], np.int32)
        Ly.intr, Ly.Tcb, Ly.has_Tcb = self.intr, self.Tcb, self.T_cb is not None
        # pixel coordinates: implicit grid when every keyframe shares one exact grid
        mode, grid = L.PIX_GRID, None
        if any(e.pixels is not None for e in self.edges):
            mode = L.PIX_EDGE
        else:
            for k in kids:
                g = self.kfs[k].grid
                if g is None or (grid is not None and g != grid):
                    mode = L.PIX_KF
                    break
                grid = g
            if grid is None:
                mode = L.PIX_KF
        Ly.mode, Ly.grid = mode, (grid if mode == L.PIX_GRID else None)
        if mode == L.PIX_KF:
            Ly.pix = np.zeros((Ly.n_disp_pad, 2), np.float32)
            for n, k in enumerate(kids):
                Ly.pix[Ly.doff_pad[n]:Ly.doff_pad[n] + npix[n]] = self.kfs[k].pixels
        elif mode == L.PIX_EDGE:
            Ly.pix = np.zeros((Ly.n_rows_pad, 2), np.float32)
            for slot, q in enumerate(order):
                e = self.edges[q]
                px = e.pixels if e.pixels is not None else self.kfs[e.i].pixels
                Ly.pix[Ly.eoff_pad[slot]:Ly.eoff_pad[slot] + len(px)] = px
        else:
            Ly.pix = None
        Ly.kids = kids
        return Ly

    def _key(self, Ly, o):
        h = hashlib.blake2b(digest_size=16)
        for a in (Ly.npix, Ly.ei, Ly.ej, Ly.fi, Ly.fj, Ly.frozen, Ly.intr, Ly.Tcb):
            h.update(np.ascontiguousarray(a).tobytes())
            h.update(b"|")
        if Ly.pix is not None:
            h.update(Ly.pix.tobytes())
        # the frozen set enters as the per-keyframe flags hashed above (kids change as a window slides)
        opts = tuple(sorted((k, tuple(v) if isinstance(v, (list, tuple)) else v) for k, v in o.items()
                            if k != "frozen_keyframes"))
        return (Ly.K, Ly.E, Ly.F, Ly.mode, Ly.grid, Ly.has_Tcb, opts, h.hexdigest())

    def _pack_into(self, Ly, tgt, w, disp64):
        """Device-to-device gather of the window into the packed solver layout (one
        vba_copy_segments launch; padding rows weight 0, padding disparities 1)."""
        w.zero_()
        tgt.zero_()
        disp64.fill_(1.0)
        segs = []
        tp, wp, dp = tgt.data_ptr(), w.data_ptr(), disp64.data_ptr()
        for slot, q in enumerate(Ly.order):
            e = self.edges[q]
            o = 8 * int(Ly.eoff_pad[slot])   # 2 floats per row
            nb = 4 * e.flow.numel()
            segs.append((e.flow.data_ptr(), tp + o, nb))
            segs.append((e.w.data_ptr(), wp + o, nb))
        for n, k in enumerate(Ly.kids):
            kf = self.kfs[k]
            segs.append((kf.disp.data_ptr(), dp + 8 * int(Ly.doff_pad[n]), 8 * kf.n))
        _segments(segs, self.device, self._stage)

    def solve(self, opts=None, use_inertial=True) -> SolveReport:
        """``solve_vi_ba`` on the window (the tracker's per-keyframe solve, frontend.py:435-450:
        ``SolveOptions(max_iterations=4, frozen_keyframes=(first kid,))``; before the inertial
        initialisation the tracker solves the vision-only shadow graph: ``use_inertial=False``
        with ``optimize_velocity_bias=False``)."""
        from .problem import options_dict
        if opts is None:
            opts = SolveOptions(max_iterations=4, frozen_keyframes=(next(iter(self.kfs)),))
        o = options_dict(opts)
        Ly = self._layout(o, use_inertial)
        key = self._key(Ly, o)
        dp = self._cache.pop(key, None)
        dev = self.device
        if dp is not None:
            dp.stream.wait_stream(torch.cuda.current_stream(dev))   # the staged insert copies
            with torch.cuda.stream(dp.stream):
                self._pack_into(Ly, dp.d_tgt, dp.d_w, dp.d_disp64)
            Ly.tgt, Ly.w, Ly.disp64 = dp.d_tgt, dp.d_w, dp.d_disp64
            dp.rebind(Ly)
        else:
            Ly.tgt = torch.empty(2 * Ly.n_rows_pad, dtype=torch.float32, device=dev)
            Ly.w = torch.empty(2 * Ly.n_rows_pad, dtype=torch.float32, device=dev)
            Ly.disp64 = torch.empty(Ly.n_disp_pad, dtype=torch.float64, device=dev)
            self._pack_into(Ly, Ly.tgt, Ly.w, Ly.disp64)
            dp = DeviceProblem(None, o, layout=Ly)
            self.replans += 1
        self._cache[key] = dp
        while len(self._cache) > self.cache_size:
            self._cache.popitem(last=False)[1].close()
        rep = dp.solve()
        self.solves += 1
        if rep["iterations"] > 0:
            L.check(dp.lib.vba_download(dp.ctx, dp._sptr()))
            with torch.cuda.stream(dp.stream):   # solved disparities stay on the device
                base = dp.d_disp64.data_ptr()
                _segments([(base + 8 * int(Ly.doff_pad[n]), self.kfs[k].disp.data_ptr(), 8 * self.kfs[k].n)
                           for n, k in enumerate(Ly.kids)], dev, self._stage)
            st = dp.d_state.cpu().numpy()
            for n, k in enumerate(Ly.kids):
                if not Ly.frozen[n]:
                    self.kfs[k].state = st[n].copy()
            if opts.optimize_gravity:
                self.grav = dp.d_grav.cpu().numpy().copy()
        self._stage.recycle()
        return SolveReport(rep["iterations"], rep["initial_cost"], rep["final_cost"], rep["cost_trajectory"],
                           rep["termination"], rep["condition_warnings"])

    # ---- interop ----------------------------------------------------------------------
    def state(self, kid):
        return self.kfs[kid].state.copy()

    def disparities(self, kid):
        return self.kfs[kid].disp.cpu().numpy()

    def graph(self):
        """The window as a host FrameGraph (paper_2512_02293_b200.types): downloads disparities."""
        from . import types as T
        kfs = []
        for k, kf in self.kfs.items():
            s = kf.state
            st = T.PoseState(T.Pose(T.Rotation(s[0:4]), s[4:7]), s[7:10], T.BiasState(s[10:13], s[13:16]), kf.ts)
            kfs.append(T.Keyframe(k, st, kf.pixels.copy(), kf.disp.cpu().numpy()))
        edges = []
        for e in self.edges:
            px = e.pixels if e.pixels is not None else self.kfs[e.i].pixels
            flow = e.flow.cpu().numpy().astype(float).reshape(-1, 2)
            edges.append(T.VisionEdge(e.i, e.j, px.copy(), px + flow, e.w.cpu().numpy().astype(float).reshape(-1, 2)))
        return kfs, edges

    @classmethod
    def from_tracker_dict(cls, data, window_size=None, device=None):
        """Replay a window serialised by the reference's ``TrackerState.to_dict``
        (frontend.py:209-294): keyframes, correspondence edges, inertial factors, gravity,
        intrinsics and extrinsic.  Quaternions are taken bit-exactly (frontend.py:565-573)."""
        from . import types as T
        gd = data["graph"]

        def rot(q):
            r = T.Rotation.identity()
            r.q = np.asarray(q, dtype=float).reshape(4)
            return r

        def pose(d):
            return T.Pose(rot(d["q"]), np.array(d["t"]))

        grav = T.GravityModel(rot(gd["gravity"]["q"]), gd["gravity"]["magnitude"])
        intr = T.Intrinsics(**gd["intrinsics"])
        T_cb = None if gd["T_cb"] is None else pose(gd["T_cb"])
        ws = window_size or data.get("policy", {}).get("window_size", 12)
        w = cls(intr, grav, T_cb, window_size=ws, device=device)
        for k in gd["keyframes"]:
            s = k["state"]
            st = T.PoseState(pose(s["pose"]), np.array(s["velocity"]),
                             T.BiasState(np.array(s["gyro_bias"]), np.array(s["accel_bias"])), s["timestamp"])
            w.add_keyframe(k["kid"], st, np.array(k["pixels"]), np.array(k["disparities"]))
        for e in gd["vision_edges"]:
            w.add_vision_edge(e["i"], e["j"], np.array(e["pixels"]), np.array(e["targets"]), np.array(e["weights"]))
        for i, j, d in gd["inertial_edges"]:
            delta = T.PreintegratedDelta(
                dt_total=d["dt_total"], delta_R=rot(d["q"]), delta_p=np.array(d["delta_p"]),
                delta_v=np.array(d["delta_v"]), J_rot=np.array(d["J_rot"]), J_pos=np.array(d["J_pos"]),
                J_vel=np.array(d["J_vel"]), covariance=np.array(d["covariance"]),
                bias_lin_point=T.BiasState(np.array(d["gyro_bias"]), np.array(d["accel_bias"])))
            w.add_inertial_edge(i, j, delta)
        w.phase = data.get("phase")
        w.solve_iterations = data.get("solve_iterations", 4)
        return w

    def close(self):
        while self._cache:
            self._cache.popitem()[1].close()
