"""Batched IMU preintegration on the GPU.

Drop-in for vislam/imu.py:77-167 (`preintegrate(samples, bias_hat, noise)`): the
same midpoint scheme, bias Jacobians and 15x15 covariance, computed by the
`vba_preintegrate` kernel (csrc/vba_preint.cu) for every keyframe pair of a
window at once instead of one Python loop per pair.  Invalid pairs raise
ValueError exactly where the reference does (imu.py:87-91).  There is no CPU
path: without the built extension or a CUDA device the calls fail.
"""

from __future__ import annotations

import importlib

import numpy as np

from . import _lib

# offsets of the fields in one output record (include/vba.h, VBA_PREINT_REC)
_LAYOUT = (("dt_total", 0, ()), ("delta_q", 1, (4,)), ("delta_p", 5, (3,)), ("delta_v", 8, (3,)),
           ("J_rot", 11, (3, 3)), ("J_pos", 20, (3, 6)), ("J_vel", 38, (3, 6)), ("covariance", 56, (15, 15)))


def _noise_vector(noise):
    if hasattr(noise, "gyro_noise_density"):
        return np.array([noise.gyro_noise_density, noise.accel_noise_density,
                         noise.gyro_bias_random_walk, noise.accel_bias_random_walk], dtype=np.float64)
    v = np.asarray(noise, dtype=np.float64).reshape(-1)
    if v.shape[0] != 4:
        raise ValueError("noise must hold (gyro, accel, gyro random walk, accel random walk) densities")
    return v


def scratch_for(n_samples, device="cuda"):
    """Reusable device workspace for preintegrate_device (vba_preint_scratch_bytes)."""
    import torch

    return torch.empty(int(_lib.load().vba_preint_scratch_bytes(int(n_samples))), dtype=torch.uint8, device=device)


def preintegrate_device(ts, gyro, accel, soff, bias, noise, out=None, scratch=None, stream=None):
    """Device-resident form: torch CUDA fp64 tensors ts [S], gyro/accel [S,3],
    soff int64 [F+1] (pair f owns samples soff[f]..soff[f+1]-1), bias [F,6],
    noise [4].  Returns (or fills) out [F, PREINT_REC]; `scratch` (scratch_for(S))
    may be kept across calls."""
    import torch

    lib = _lib.load()
    F = int(soff.shape[0]) - 1
    dev = ts.device
    S = int(ts.shape[0])
    if out is None:
        out = torch.empty((max(F, 0), _lib.PREINT_REC), dtype=torch.float64, device=dev)
    if scratch is None or scratch.numel() < lib.vba_preint_scratch_bytes(S):
        scratch = scratch_for(S, dev)
    st = (stream or torch.cuda.current_stream(dev)).cuda_stream
    rc = lib.vba_preintegrate(ts.data_ptr(), gyro.data_ptr(), accel.data_ptr(), S, soff.data_ptr(), F,
                              bias.data_ptr(), noise.data_ptr(), scratch.data_ptr(), out.data_ptr(), st)
    if rc == _lib.VBA_E_INVALID:
        raise ValueError(lib.vba_last_error().decode())
    _lib.check(rc)
    return out


def factor_records(rec, bias, out=None, stream=None):
    """Device [F, PREINT_REC] records + bias linearisation points [F, 6] -> the solver's
    IMU factor records [F, IMU_REC] (vba_preint_factor_records), on the device: feed them
    to DeviceProblem.d_imu / a solve_windows window without a host round trip."""
    import torch

    lib = _lib.load()
    F = int(rec.shape[0])
    if out is None:
        out = torch.empty((F, _lib.IMU_REC), dtype=torch.float64, device=rec.device)
    st = (stream or torch.cuda.current_stream(rec.device)).cuda_stream
    _lib.check(lib.vba_preint_factor_records(rec.data_ptr(), bias.data_ptr(), F, out.data_ptr(), st))
    return out


def unpack(rec):
    """Split [F, PREINT_REC] records into a dict of per-field arrays ([F, ...])."""
    rec = np.asarray(rec)
    F = rec.shape[0]
    d = {}
    for name, off, shape in _LAYOUT:
        n = int(np.prod(shape)) if shape else 1
        d[name] = rec[:, off:off + n].reshape((F,) + shape) if shape else rec[:, off].copy()
    return d


def preintegrate_batch(ts_list, gyro_list, accel_list, bias, noise, device="cuda"):
    """Preintegrate F keyframe pairs on the GPU.  ts_list[f] [S_f], gyro_list[f] /
    accel_list[f] [S_f, 3], bias [F, 6] (gyro bias, accel bias), noise = an
    ImuNoiseModel-like object or (gyro, accel, gyro rw, accel rw).  Returns a dict
    of fp64 arrays: dt_total [F], delta_q [F,4] (wxyz, w >= 0), delta_p, delta_v
    [F,3], J_rot [F,3,3], J_pos, J_vel [F,3,6], covariance [F,15,15]."""
    import torch

    F = len(ts_list)
    if len(gyro_list) != F or len(accel_list) != F:
        raise ValueError("ts, gyro and accel lists must have one entry per pair")
    bias = np.ascontiguousarray(np.asarray(bias, dtype=np.float64).reshape(F, 6))
    ts = [np.asarray(t, dtype=np.float64).reshape(-1) for t in ts_list]
    gy = [np.asarray(g, dtype=np.float64).reshape(-1, 3) for g in gyro_list]
    ac = [np.asarray(a, dtype=np.float64).reshape(-1, 3) for a in accel_list]
    for t, g, a in zip(ts, gy, ac):
        if g.shape[0] != t.shape[0] or a.shape[0] != t.shape[0]:
            raise ValueError("each sample needs a timestamp, a gyro and an accel reading")
    soff = np.zeros(F + 1, dtype=np.int64)
    soff[1:] = np.cumsum([t.shape[0] for t in ts])
    cat = (lambda xs, w: np.concatenate(xs) if F else np.zeros((0,) + w))
    host = [cat(ts, ()), cat(gy, (3,)), cat(ac, (3,)), soff, bias, _noise_vector(noise)]
    dev = [torch.from_numpy(np.ascontiguousarray(h)).to(device) for h in host]
    out = preintegrate_device(*dev)
    return unpack(out.cpu().numpy())


def preintegrate(samples, bias_hat, noise):
    """Reference signature (imu.py:77): `samples` = ImuSample-like objects
    (timestamp, gyro, accel), `bias_hat` = BiasState-like, `noise` =
    ImuNoiseModel-like.  Returns the caller's PreintegratedDelta type (found in
    the module that defines type(bias_hat)) when it exists, else the field dict."""
    d = preintegrate_many([(samples, bias_hat)], noise)
    return d[0]


def preintegrate_many(pairs, noise):
    """All keyframe pairs of a window in one launch: `pairs` = [(samples, bias_hat)]."""
    ts = [[s.timestamp for s in smp] for smp, _ in pairs]
    gy = [[s.gyro for s in smp] for smp, _ in pairs]
    ac = [[s.accel for s in smp] for smp, _ in pairs]
    for t in ts:
        if len(t) < 2:
            raise ValueError("Need at least two IMU samples to preintegrate")
    bias = np.array([np.concatenate([b.gyro_bias, b.accel_bias]) for _, b in pairs], dtype=np.float64)
    r = preintegrate_batch(ts, gy, ac, bias.reshape(len(pairs), 6), noise)
    res = []
    for f, (_, b) in enumerate(pairs):
        fields = {k: r[k][f] for k, _, _ in _LAYOUT}
        mod = importlib.import_module(type(b).__module__)
        Delta, Rot = getattr(mod, "PreintegratedDelta", None), getattr(mod, "Rotation", None)
        if Delta is None or Rot is None:
            res.append(fields)
            continue
        res.append(Delta(dt_total=float(fields["dt_total"]), delta_R=Rot(fields["delta_q"]),
                         delta_p=fields["delta_p"], delta_v=fields["delta_v"], J_rot=fields["J_rot"],
                         J_pos=fields["J_pos"], J_vel=fields["J_vel"], covariance=fields["covariance"],
                         bias_lin_point=b.copy()))
    return res
