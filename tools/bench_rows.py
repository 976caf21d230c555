"""Measurements of the SURVEY §8(f) rows beside the VI-BA bench (one JSON line each).

* pgba   -- Sim(3) pose-graph BA on make_pgba_workload() (256 nodes, 8 dense 48x64 loop edges,
            255 chain factors, 6 LM iterations): device-resident GPU solve (CUDA events) vs the
            CPU reference restatement (oracle/pgba.py, fp64 numpy) on the same graph;
* window -- the tracker's per-keyframe window solve (12-keyframe window, covisibility radius 3,
            48x64 pixels, 4 LM iterations) through window.DeviceWindow in the steady state
            (insert keyframe + edges + IMU factor, solve, evict), wall clock per keyframe,
            vs the drop-in solver.solve_vi_ba on the same host graph and vs the CPU reference;
* init   -- stage-2 inertial-only initialisation (initialization.init_inertial_only) on a
            20-keyframe window vs the CPU reference restatement (oracle/init.py).

python tools/bench_rows.py [pgba window init]
"""
import copy
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def ev_time(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def bench_pgba():
    import oracle.pgba as O
    from paper_2512_02293_b200.pgba import DevicePoseGraph, pack_pose_graph
    from paper_2512_02293_b200.workloads import make_pgba_workload
    g, _ = make_pgba_workload()
    P = pack_pose_graph(g)
    opts = {"max_iterations": 6}
    DevicePoseGraph(copy.deepcopy(P), opts).solve()   # warm-up (module load, allocator)
    ms_list = []
    for _ in range(5):
        dp2 = DevicePoseGraph(copy.deepcopy(P), opts)
        ms, rep = ev_time(dp2.solve, 1)
        ms_list.append(ms)
        dp2.close()
    ms = float(np.median(ms_list))
    px = int(P["veoff"][-1])
    Q = copy.deepcopy(P)
    t0 = time.perf_counter()
    ro = O.solve_pgba(Q, opts)
    cpu_s = time.perf_counter() - t0
    return {"row": "pgba", "workload": "make_pgba_workload(): 256 Sim(3) nodes, 8 loop edges x 3072 px, 255 chain factors",
            "gpu_ms_per_solve": ms, "iterations": rep["iterations"],
            "gpu_iterations_per_s": rep["iterations"] / (ms / 1e3),
            "gpu_loop_px_per_s": px * rep["iterations"] / (ms / 1e3),
            "cpu_reference_s": cpu_s, "cpu_iterations": ro["iterations"], "cpu_kind": "port (oracle/pgba.py, fp64 numpy)",
            "speedup": cpu_s / (ms / 1e3), "final_cost_gpu": rep["final_cost"], "final_cost_cpu": ro["final_cost"]}


def bench_window():
    import oracle
    from paper_2512_02293_b200 import solver as S
    from paper_2512_02293_b200 import types as T
    from paper_2512_02293_b200.problem import pack_graph
    from paper_2512_02293_b200.types import SolveOptions
    from paper_2512_02293_b200.window import DeviceWindow
    from paper_2512_02293_b200.workloads import make_workload
    g = make_workload(3)          # 128 keyframes of 48x64: the stream
    W, R = 12, 3
    by_pair = {(e.i, e.j): e for e in g.vision_edges}
    win = DeviceWindow(g.intrinsics, g.gravity, None, window_size=W)
    h_kfs, h_edges, h_imu = [], [], []
    t_win, t_drop, t_cpu, h2d, last_graph = [], [], [], [], None
    for k in range(48):
        kf = g.keyframes[k]
        t0 = time.perf_counter()
        b0 = win.h2d_bytes
        win.add_keyframe(k, kf.state, kf.pixels, kf.disparities)
        live = list(win.kfs)
        new_edges = []
        for n in live[-(R + 1):-1]:
            for (i, j) in ((k, n), (n, k)):
                e = by_pair.get((i, j))
                if e is not None:
                    win.add_vision_edge(i, j, e.pixels, e.targets, e.weights)
                    new_edges.append(e)
        if k > 0:
            win.add_inertial_edge(*g.inertial_edges[k - 1])
        opts = SolveOptions(max_iterations=4, frozen_keyframes=(live[0],))
        if len(live) >= 2:
            win.solve(opts)
        win.evict_to_size()
        torch.cuda.synchronize()
        t_win.append(time.perf_counter() - t0)
        h2d.append(win.h2d_bytes - b0)
        # the same window through the drop-in (host graph rebuilt like the reference's tracker)
        h_kfs.append(T.Keyframe(k, kf.state.copy(), kf.pixels, kf.disparities.copy()))
        h_edges += [T.VisionEdge(e.i, e.j, e.pixels, e.targets, e.weights) for e in new_edges]
        if k > 0:
            h_imu.append(g.inertial_edges[k - 1])
        t0 = time.perf_counter()
        hg = T.FrameGraph(list(h_kfs), list(h_edges), list(h_imu), g.gravity, g.intrinsics)
        if len(h_kfs) >= 2:
            S.solve_vi_ba(hg, SolveOptions(max_iterations=4, frozen_keyframes=(h_kfs[0].kid,)))
        torch.cuda.synchronize()
        t_drop.append(time.perf_counter() - t0)
        last_graph = hg
        while len(h_kfs) > W:
            old = h_kfs.pop(0).kid
            h_edges = [e for e in h_edges if e.i != old and e.j != old]
            h_imu = [t for t in h_imu if t[0] != old]
    # CPU reference on a full steady-state window (bounded sample: 3 windows)
    P = pack_graph(last_graph)
    for _ in range(3):
        t0 = time.perf_counter()
        oracle.solve_vi_ba(copy.deepcopy(P), {"max_iterations": 4, "frozen_keyframes": (int(P["kid"][0]),)})
        t_cpu.append(time.perf_counter() - t0)
    steady = slice(20, None)
    epx = int(sum(len(e.pixels) for e in last_graph.vision_edges))
    return {"row": "window", "workload": f"tracker stream over config 3's keyframes: window {W}, covisibility radius {R}, "
                                         f"48x64 px, 4 LM iterations ({epx} edge-px per window)",
            "device_window_ms_per_keyframe": 1e3 * float(np.median(np.array(t_win)[steady])),
            "dropin_ms_per_keyframe": 1e3 * float(np.median(t_drop[steady])),
            "cpu_reference_ms_per_keyframe": 1e3 * float(np.median(t_cpu)),
            "cpu_kind": "port (oracle/vi_ba.py, fp64 numpy)",
            "h2d_bytes_per_keyframe": int(np.median(np.array(h2d)[steady])),
            "plans": win.replans, "solves": win.solves,
            "speedup_vs_cpu": float(np.median(t_cpu) / np.median(np.array(t_win)[steady]))}


def bench_init():
    import oracle.init as OI
    from paper_2512_02293_b200.initialization import init_inertial_only
    from paper_2512_02293_b200.problem import pack_graph
    from paper_2512_02293_b200.workloads import make_workload
    g = make_workload(3)
    g.keyframes = g.keyframes[:20]
    g.vision_edges = [e for e in g.vision_edges if e.i < 20 and e.j < 20]
    g.inertial_edges = g.inertial_edges[:19]
    for _ in range(3):   # module load, allocator pools
        init_inertial_only(g)
    torch.cuda.synchronize()
    ts = []
    for _ in range(21):  # median of 21 calls: single calls see host-side spikes of 10-40 ms
        t0 = time.perf_counter()
        res = init_inertial_only(g)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    P = pack_graph(g)
    t0 = time.perf_counter()
    s, _, _, _, rep = OI.init_inertial_only(P)
    cpu = time.perf_counter() - t0
    return {"row": "init", "workload": "stage-2 inertial-only initialisation, 20 keyframes of config 3 (69 unknowns)",
            "gpu_ms": 1e3 * float(np.median(ts)), "gpu_iterations": res.reports["inertial"].iterations,
            "cpu_reference_ms": 1e3 * cpu, "cpu_iterations": rep["iterations"], "cpu_kind": "port (oracle/init.py)",
            "log_scale_gpu": res.log_scale, "log_scale_cpu": s, "speedup": cpu / float(np.median(ts))}


if __name__ == "__main__":
    which = sys.argv[1:] or ["pgba", "window", "init"]
    for w in which:
        print(json.dumps({"pgba": bench_pgba, "window": bench_window, "init": bench_init}[w]()), flush=True)
