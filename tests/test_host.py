"""Host-side logic (no GPU): packing, validation, device layout, write-back, workloads."""
import copy

import numpy as np
import pytest

from conftest import graph_from_packed, load_golden
from paper_2512_02293_b200 import _lib as L
from paper_2512_02293_b200 import types as T
from paper_2512_02293_b200.device import HostLayout, detect_pixel_mode, imu_records
from paper_2512_02293_b200.problem import pack_graph, write_back
from paper_2512_02293_b200.workloads import CONFIGS, make_workload


def test_pack_roundtrip_equals_golden_inputs():
    P, _, _ = load_golden("win8_px30")
    g = graph_from_packed(P)
    Q = pack_graph(g)
    for k in ("q", "p", "v", "bg", "ba", "disp", "pix", "ei", "ej", "eoff", "tgt", "w", "f_cov", "f_bhat"):
        assert np.array_equal(np.asarray(Q[k]), np.asarray(P[k])), k


def test_validation_mirrors_reference_errors():
    P, _, _ = load_golden("win4_tcb")
    g = graph_from_packed(P)
    bad = copy.deepcopy(g)
    e = bad.vision_edges[0]
    bad.vision_edges[0] = T.VisionEdge(e.i, e.j, e.pixels[:-1], e.targets[:-1], e.weights[:-1])
    with pytest.raises(ValueError):                      # residuals.py:181-183
        pack_graph(bad)
    bad = copy.deepcopy(g)
    bad.keyframes[1].state.timestamp += 0.5               # residuals.py:281-284
    with pytest.raises(ValueError):
        pack_graph(bad)
    with pytest.raises(ValueError):                       # solver.py:70-73
        T.FrameGraph(g.keyframes, g.vision_edges, g.inertial_edges[:-1], g.gravity, g.intrinsics)
    with pytest.raises(ValueError):
        T.VisionEdge(0, 1, np.zeros((2, 2)), np.zeros((2, 2)), -np.ones((2, 2)))
    with pytest.raises(ValueError):
        T.Keyframe(0, g.keyframes[0].state, np.zeros((1, 2)), np.array([0.0]))


def test_host_layout_sorted_padded_flow():
    P, _, opts = load_golden("win6_frozen2")
    H = HostLayout(P, opts)
    assert np.all(np.diff(H.ei) >= 0)                    # sorted by source
    assert np.all(H.doff_pad % 4 == 0) and np.all(H.eoff_pad % 4 == 0)
    assert H.mode == L.PIX_KF                             # random sub-pixel coordinates
    # flow rows = targets - source pixels, in the stable source order
    for k, e in enumerate(H.edge_order):
        r0, r1 = P["eoff"][e], P["eoff"][e + 1]
        want = (P["tgt"][r0:r1] - P["epix"][r0:r1]).astype(np.float32)
        got = H.tgt[H.eoff_pad[k]:H.eoff_pad[k] + (r1 - r0)]
        assert np.array_equal(got, want)
        assert np.all(H.w[H.eoff_pad[k] + (r1 - r0):H.eoff_pad[k] + ((r1 - r0 + 3) // 4) * 4] == 0)
    assert H.frozen.tolist() == [int(k in (0, 3)) for k in P["kid"]]


def test_pixel_mode_detection():
    P = pack_graph(make_workload(0, grid=(6, 8)))
    mode, gp = detect_pixel_mode(P)
    assert mode == L.PIX_GRID and gp == (0.0, 0.0, 1.0, 1.0, 8)
    Q = copy.deepcopy(P)
    Q["epix"] = Q["epix"] + 0.25                          # edges disagree with keyframe pixels
    assert detect_pixel_mode(Q)[0] == L.PIX_EDGE


def test_imu_record_layout():
    P, _, _ = load_golden("win5_gravity")
    R = imu_records(P)
    assert R.shape == (len(P["fi"]), L.IMU_REC)
    assert np.array_equal(R[:, 56:137].reshape(-1, 9, 9), P["f_cov"][:, :9, :9])
    assert np.array_equal(R[:, 137:173].reshape(-1, 6, 6), P["f_cov"][:, 9:15, 9:15])


def test_write_back_semantics():
    P, _, _ = load_golden("win5_gravity")
    g = graph_from_packed(P)
    frozen_state = g.keyframes[0].state
    other = g.keyframes[1].state
    K = len(g.keyframes)
    q = np.tile([1.0, 0, 0, 0], (K, 1))
    opts = T.SolveOptions(optimize_gravity=True)
    write_back(g, q, np.ones((K, 3)), np.zeros((K, 3)), np.zeros((K, 3)), np.zeros((K, 3)),
               np.full(len(P["disp"]), 0.5), np.array([1.0, 0, 0, 0]), opts)
    assert g.keyframes[0].state is frozen_state          # gauge keyframe untouched
    assert g.keyframes[1].state is not other
    assert np.all(g.keyframes[1].state.pose.translation == 1.0)
    assert np.all(g.keyframes[0].disparities == 0.5)      # disparities never frozen


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_workload_shapes_match_baseline(cfg):
    spec = CONFIGS[cfg]
    g = make_workload(cfg)
    assert len(g.keyframes) == spec.n_kf
    assert len(g.vision_edges) == spec.n_edges
    assert len(g.inertial_edges) == spec.n_kf - 1
    assert all(len(kf.disparities) == spec.grid[0] * spec.grid[1] for kf in g.keyframes)
    loops = sum(abs(e.i - e.j) > 30 for e in g.vision_edges)
    assert loops == spec.n_loop
    assert all(np.all(e.weights >= 0) and np.all(e.weights <= 1) for e in g.vision_edges)


def test_workload_is_seeded():
    a, b = pack_graph(make_workload(1)), pack_graph(make_workload(1))
    for k in ("q", "p", "disp", "tgt", "w", "f_dp"):
        assert np.array_equal(a[k], b[k])


def test_bench_bounded_sample():
    import bench
    P = pack_graph(make_workload(3))
    Q, M, epx = bench.bounded_sample(P, 300_000)
    assert epx >= 300_000 and M < len(P["kid"])
    assert np.all(Q["ei"] < M) and np.all(Q["ej"] < M)
    assert Q["eoff"][-1] == len(Q["tgt"]) == epx


_LAYOUT_FIELDS = ("npix", "doff_pad", "edge_order", "eoff_pad", "tgt", "w", "dsrc", "disp", "ei", "ej", "fi", "fj",
                  "imu", "state", "ts", "grav", "frozen", "intr", "Tcb")


@pytest.mark.parametrize("name", ["win6_frozen2", "win4_tcb", "win5_gravity", "cfg0_grid12x16", "edge_pixels",
                                  "workload1"])
def test_graph_layout_equals_packed_layout(name):
    """HostLayout.from_graph (native packer, csrc/vba_pack.cpp) is bitwise the packed-dict layout."""
    if name == "workload1":
        g = make_workload(1)
        opts = {"frozen_keyframes": (0,)}
    else:
        P, _, opts = load_golden("win8_px30" if name == "edge_pixels" else name)
        g = graph_from_packed(P)
        if name == "edge_pixels":          # an edge whose pixels differ from its keyframe's: VBA_PIX_EDGE
            e = g.vision_edges[3]
            g.vision_edges[3] = T.VisionEdge(e.i, e.j, e.pixels + 0.5, e.targets, e.weights)
    H1 = HostLayout(pack_graph(g), opts)
    H2 = HostLayout.from_graph(g, opts, pinned=False)
    for k in _LAYOUT_FIELDS:
        assert np.array_equal(getattr(H1, k), getattr(H2, k)), k
    assert H1.mode == H2.mode and H1.grid == H2.grid
    assert (H1.pix is None) == (H2.pix is None) and (H1.pix is None or np.array_equal(H1.pix, H2.pix))
    if name == "edge_pixels":
        assert H2.mode == L.PIX_EDGE
    if name == "workload1":
        assert H2.mode == L.PIX_GRID


def test_graph_layout_validation():
    """from_graph raises the reference's ValueErrors (residuals.py:181-185, 112-113, 281-284)."""
    P, _, opts = load_golden("win4_tcb")
    g = graph_from_packed(P)
    bad = copy.deepcopy(g)
    e = bad.vision_edges[0]
    bad.vision_edges[0] = T.VisionEdge(e.i, e.j, e.pixels[:-1], e.targets[:-1], e.weights[:-1])
    with pytest.raises(ValueError):
        HostLayout.from_graph(bad, opts, pinned=False)
    bad = copy.deepcopy(g)
    bad.vision_edges[1].weights = -bad.vision_edges[1].weights - 1.0      # mutated after construction
    with pytest.raises(ValueError):
        HostLayout.from_graph(bad, opts, pinned=False)
    bad = copy.deepcopy(g)
    bad.keyframes[1].state.timestamp += 0.5
    with pytest.raises(ValueError):
        HostLayout.from_graph(bad, opts, pinned=False)
    bad = copy.deepcopy(g)
    bad.keyframes[2].disparities = bad.keyframes[2].disparities * 0.0
    with pytest.raises(ValueError):
        HostLayout.from_graph(bad, opts, pinned=False)
