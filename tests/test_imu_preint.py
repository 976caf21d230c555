"""IMU preintegration (reference vislam/imu.py:77-167).

CPU: the oracle restatement against the reference's own outputs (tests/golden/imu/imu_preint.npz,
made by tests/golden/make_imu_golden.py).  GPU: the batched device kernel
(`vba_preintegrate`, one thread per keyframe pair) against the same goldens, and its errors."""
import os

import numpy as np
import pytest

from oracle.imu import preintegrate as oracle_preintegrate

HERE = os.path.dirname(os.path.abspath(__file__))
FIELDS = ("delta_q", "delta_p", "delta_v", "J_rot", "J_pos", "J_vel", "covariance")


def _cases():
    z = np.load(os.path.join(HERE, "golden", "imu", "imu_preint.npz"))
    return z["noise"], [{k[len(f"c{i}_"):]: z[k] for k in z.files if k.startswith(f"c{i}_")}
                        for i in range(int(z["n"]))]


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    s = max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / s)


def test_oracle_matches_reference_goldens():
    noise, cases = _cases()
    for c in cases:
        d = oracle_preintegrate(c["ts"], c["gyro"], c["accel"], c["bias"], noise)
        assert abs(d["dt_total"] - float(c["dt_total"])) <= 1e-15
        for f in FIELDS:
            assert _rel(d[f], c[f]) < 1e-13, f


def test_oracle_rejects_like_reference():
    with pytest.raises(ValueError):
        oracle_preintegrate([0.0], np.zeros((1, 3)), np.zeros((1, 3)), np.zeros(6), (1, 1, 1, 1))
    with pytest.raises(ValueError):
        oracle_preintegrate([0.0, 0.0], np.zeros((2, 3)), np.zeros((2, 3)), np.zeros(6), (1, 1, 1, 1))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["seq", "scan"])
def test_device_preintegration_matches_reference(cuda_ok, mode, monkeypatch):
    """Both propagation kernels -- the sequential one (16 lanes per pair) and the log-depth scan
    (one warp per pair, composed affine maps; the default from 64 intervals per pair) -- against
    the reference's goldens."""
    from paper_2512_02293_b200.imu import preintegrate_batch
    monkeypatch.setenv("VBA_PREINT", mode)
    noise, cases = _cases()
    out = preintegrate_batch([c["ts"] for c in cases], [c["gyro"] for c in cases],
                             [c["accel"] for c in cases], np.stack([c["bias"] for c in cases]), noise)
    for i, c in enumerate(cases):
        assert abs(out["dt_total"][i] - float(c["dt_total"])) <= 1e-15
        for f in FIELDS:
            assert _rel(out[f][i], c[f]) < 1e-12, (i, f)


@pytest.mark.gpu
def test_device_preintegration_errors(cuda_ok):
    from paper_2512_02293_b200.imu import preintegrate_batch
    z3 = np.zeros((2, 3))
    with pytest.raises(ValueError):
        preintegrate_batch([np.array([0.0, 0.0])], [z3], [z3], np.zeros((1, 6)), (1, 1, 1, 1))
    with pytest.raises(ValueError):
        preintegrate_batch([np.array([0.0])], [z3[:1]], [z3[:1]], np.zeros((1, 6)), (1, 1, 1, 1))


@pytest.mark.gpu
def test_device_preintegration_reference_signature(cuda_ok):
    """preintegrate(samples, bias_hat, noise) with the reference's object shapes (imu.py:18-62)."""
    from types import SimpleNamespace

    from paper_2512_02293_b200.imu import preintegrate, preintegrate_batch
    noise, cases = _cases()
    c = cases[3]
    samples = [SimpleNamespace(timestamp=float(t), gyro=g, accel=a) for t, g, a in zip(c["ts"], c["gyro"], c["accel"])]
    bias = SimpleNamespace(gyro_bias=c["bias"][:3], accel_bias=c["bias"][3:])
    nm = SimpleNamespace(gyro_noise_density=noise[0], accel_noise_density=noise[1],
                         gyro_bias_random_walk=noise[2], accel_bias_random_walk=noise[3])
    d = preintegrate(samples, bias, nm)
    for f in FIELDS:
        assert _rel(d[f], c[f]) < 1e-12, f
    empty = preintegrate_batch([], [], [], np.zeros((0, 6)), noise)
    assert empty["covariance"].shape == (0, 15, 15)


@pytest.mark.gpu
def test_device_preintegration_feeds_the_solver(cuda_ok):
    """Raw IMU stream -> vba_preintegrate -> vba_preint_factor_records -> the solver's IMU
    buffer, all on the device: the records match the host packing of the workload's own
    (numpy, imu.py scheme) deltas, and a solve_windows window fed with them reaches the
    host-packed solve's cost and states."""
    import copy

    import torch

    from paper_2512_02293_b200 import _lib
    from paper_2512_02293_b200.device import DeviceProblem
    from paper_2512_02293_b200.imu import factor_records, preintegrate_device
    from paper_2512_02293_b200.problem import pack_graph
    from paper_2512_02293_b200.workloads import make_workload

    g = make_workload(1)
    ims = g.imu_stream
    idx = ims["idx"]
    F, S1 = idx.shape
    dev = "cuda"
    ts = torch.from_numpy(ims["ts"][idx].reshape(-1).copy()).to(dev)
    gy = torch.from_numpy(ims["gyro"][idx].reshape(-1, 3).copy()).to(dev)
    ac = torch.from_numpy(ims["accel"][idx].reshape(-1, 3).copy()).to(dev)
    soff = torch.arange(F + 1, dtype=torch.int64, device=dev) * S1
    bias = torch.from_numpy(ims["bias"].copy()).to(dev)
    noise = torch.tensor(ims["noise"], dtype=torch.float64, device=dev)
    rec = preintegrate_device(ts, gy, ac, soff, bias, noise)
    imu_dev = factor_records(rec, bias)
    P = pack_graph(g)
    opts = {"max_iterations": 2}
    dp = DeviceProblem(copy.deepcopy(P), opts)
    host = dp.H.imu
    got = imu_dev.cpu().numpy()
    assert got.shape == host.shape == (F, _lib.IMU_REC)
    for lo, hi in ((0, 1), (1, 5), (5, 8), (8, 11), (11, 20), (20, 38), (38, 56), (56, 137), (137, 173), (173, 179)):
        assert _rel(got[:, lo:hi], host[:, lo:hi]) < 1e-10, (lo, hi)
    H = dp.H
    win = {k: torch.from_numpy(np.ascontiguousarray(v).reshape(-1)).pin_memory()
           for k, v in (("state", H.state), ("disp", H.disp), ("tgt", H.tgt), ("w", H.w), ("grav", H.grav))}
    ref_rep = dp.solve_windows([dict(win, imu=torch.from_numpy(host.reshape(-1).copy()).pin_memory())])[0]
    ref_state = dp.download()
    rep = dp.solve_windows([dict(win, imu=imu_dev.reshape(-1))])[0]
    st = dp.download()
    assert abs(rep["final_cost"] - ref_rep["final_cost"]) <= 1e-9 * abs(ref_rep["final_cost"])
    for k in ref_state:
        a, b = np.asarray(st[k], float), np.asarray(ref_state[k], float)
        assert np.abs(a - b).max(initial=0.0) <= 1e-8 * max(1.0, np.abs(b).max(initial=0.0)), k


def test_record_layout_and_noise_parsing():
    """Host side of paper_2512_02293_b200.imu (no GPU): the record layout covers
    VBA_PREINT_REC exactly, unpack() splits it per field, noise objects / tuples parse."""
    from types import SimpleNamespace

    from paper_2512_02293_b200 import _lib
    from paper_2512_02293_b200.imu import _LAYOUT, _noise_vector, unpack
    end = 0
    for _, off, shape in _LAYOUT:
        assert off == end
        end = off + int(np.prod(shape)) if shape else off + 1
    assert end == _lib.PREINT_REC
    rec = np.arange(2 * _lib.PREINT_REC, dtype=float).reshape(2, -1)
    d = unpack(rec)
    assert d["dt_total"].tolist() == [0.0, float(_lib.PREINT_REC)]
    assert d["covariance"].shape == (2, 15, 15) and d["covariance"][1, 0, 0] == _lib.PREINT_REC + 56
    assert d["J_pos"][0, 2, 5] == 20 + 17
    nm = SimpleNamespace(gyro_noise_density=1.0, accel_noise_density=2.0, gyro_bias_random_walk=3.0,
                         accel_bias_random_walk=4.0)
    assert _noise_vector(nm).tolist() == [1.0, 2.0, 3.0, 4.0]
    assert _noise_vector((1, 2, 3, 4)).tolist() == [1.0, 2.0, 3.0, 4.0]
    with pytest.raises(ValueError):
        _noise_vector((1, 2, 3))
