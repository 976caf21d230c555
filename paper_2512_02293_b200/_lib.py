"""ctypes binding of the C ABI in include/vba.h (libvba = ``_vba.so``, built in-tree).

There is no fallback: if the shared library is missing, or no CUDA device is
present, calls fail loudly (``VbaError`` / ``RuntimeError``).
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VBA_LIB") or os.path.join(HERE, "_vba.so")   # VBA_LIB: tuning builds (tools/)

VBA_OK, VBA_E_INVALID, VBA_E_CUDA, VBA_E_NOT_SPD, VBA_E_COV, VBA_E_UNSUPPORTED, VBA_E_NONFINITE = range(7)
PG_REL_REC = 64
PIX_GRID, PIX_KF, PIX_EDGE = 0, 1, 2
IMU_REC = 180
PREINT_REC = 281

EXPORTED = ("vba_last_error", "vba_version", "vba_create", "vba_destroy", "vba_set_collective", "vba_set_gather",
            "vba_reduced_dim", "vba_energy", "vba_linearize", "vba_export_normal_eq",
            "vba_solve_step", "vba_export_step", "vba_export_reduced", "vba_apply_step", "vba_restore", "vba_accept",
            "vba_trial", "vba_solve", "vba_download", "vba_launch_count", "vba_stage_times",
            "vba_load_state", "vba_bind_inputs", "vba_set_profiling", "vba_stats", "vba_gram_kind", "vba_chol_plan", "vba_spd_solve", "vba_solve_times",
            "vba_preintegrate", "vba_preint_scratch_bytes",
            "vba_preint_factor_records", "vba_copy_segments",
            "vba_pg_create", "vba_pg_destroy", "vba_pg_energy", "vba_pg_linearize", "vba_pg_export_normal_eq",
            "vba_pg_solve_step", "vba_pg_export_step", "vba_pg_solve", "vba_pg_download", "vba_init_inertial")


class VbaCopySeg(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("bytes", C.c_int64)]


class VbaProblem(C.Structure):
    _fields_ = [
        ("n_kf", C.c_int32), ("n_edges", C.c_int32), ("n_imu", C.c_int32), ("pixel_mode", C.c_int32),
        ("n_disp_pad", C.c_int64), ("n_rows_pad", C.c_int64),
        ("grid_w", C.c_int32), ("has_Tcb", C.c_int32),
        ("grid_ox", C.c_double), ("grid_oy", C.c_double), ("grid_sx", C.c_double), ("grid_sy", C.c_double),
        ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
        ("Tcb", C.c_double * 7),
        ("state", C.c_void_p), ("ts", C.c_void_p), ("disp", C.c_void_p), ("pix", C.c_void_p),
        ("tgt", C.c_void_p), ("wts", C.c_void_p), ("imu", C.c_void_p), ("grav", C.c_void_p),
        ("h_doff", C.c_void_p), ("h_npix", C.c_void_p), ("h_edge_i", C.c_void_p), ("h_edge_j", C.c_void_p),
        ("h_eoff", C.c_void_p), ("h_imu_i", C.c_void_p), ("h_imu_j", C.c_void_p), ("h_frozen", C.c_void_p),
        ("disp64", C.c_void_p),
        ("shard_world", C.c_int32), ("shard_rank", C.c_int32), ("h_shard_kbounds", C.c_void_p),
    ]


class VbaPgProblem(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32), ("n_vis", C.c_int32), ("n_rel", C.c_int32), ("has_Tcb", C.c_int32),
        ("n_disp", C.c_int64), ("n_rows", C.c_int64),
        ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
        ("Tcb", C.c_double * 7),
        ("state", C.c_void_p), ("disp", C.c_void_p), ("pix", C.c_void_p), ("tgt", C.c_void_p),
        ("wts", C.c_void_p), ("rel", C.c_void_p),
        ("h_doff", C.c_void_p), ("h_npix", C.c_void_p), ("h_vis_i", C.c_void_p), ("h_vis_j", C.c_void_p),
        ("h_voff", C.c_void_p), ("h_rel_i", C.c_void_p), ("h_rel_j", C.c_void_p),
    ]


class VbaInitProblem(C.Structure):
    _fields_ = [
        ("n_kf", C.c_int32), ("n_imu", C.c_int32),
        ("q", C.c_void_p), ("p", C.c_void_p), ("v0", C.c_void_p), ("imu", C.c_void_p),
        ("h_imu_i", C.c_void_p), ("h_imu_j", C.c_void_p),
        ("grav_q", C.c_double * 4), ("grav_G", C.c_double), ("bias0", C.c_double * 6),
    ]


class VbaInitOptions(C.Structure):
    _fields_ = [("max_iterations", C.c_int32), ("damping", C.c_double)]


class VbaInitResult(C.Structure):
    _fields_ = [
        ("log_scale", C.c_double), ("grav_q", C.c_double * 4), ("bias", C.c_double * 6),
        ("iterations", C.c_int32), ("termination", C.c_int32), ("n_costs", C.c_int32),
        ("initial_cost", C.c_double), ("final_cost", C.c_double),
    ]


class VbaOptions(C.Structure):
    _fields_ = [
        ("max_iterations", C.c_int32),
        ("damping", C.c_double), ("damping_up", C.c_double), ("damping_down", C.c_double),
        ("rel_decrease_tol", C.c_double), ("step_tol", C.c_double), ("max_damping", C.c_double),
        ("optimize_gravity", C.c_int32), ("optimize_velocity_bias", C.c_int32), ("use_schur", C.c_int32),
        ("ridge", C.c_double),
    ]


class VbaReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("termination", C.c_int32), ("n_costs", C.c_int32),
        ("n_warnings", C.c_int32), ("trials", C.c_int32),
        ("initial_cost", C.c_double), ("final_cost", C.c_double),
    ]


class VbaTrialResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("new_cost", C.c_double), ("step_inf", C.c_double)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_int32, C.c_void_p)


class VbaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"vba error {code}: {msg}")
        self.code = code


_lib = None


def load(path: str | None = None):
    """Load libvba; raises if it has not been built (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"CUDA extension not built: {p} missing (run __graft_entry__.build())")
    lib = C.CDLL(p)
    v = C.c_void_p
    sig = {
        "vba_last_error": ([], C.c_char_p),
        "vba_version": ([], C.c_int),
        "vba_create": ([C.POINTER(C.c_void_p), C.POINTER(VbaProblem), C.POINTER(VbaOptions), v], C.c_int),
        "vba_destroy": ([v], C.c_int),
        "vba_set_collective": ([v, ALLREDUCE_FN, v], C.c_int),
        "vba_set_gather": ([v, ALLGATHER_FN, v], C.c_int),
        "vba_reduced_dim": ([v], C.c_int64),
        "vba_energy": ([v, v, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
        "vba_linearize": ([v, v], C.c_int),
        "vba_export_normal_eq": ([v, v, v, v, v, v, v], C.c_int),
        "vba_solve_step": ([v, v, C.c_double, C.c_int32], C.c_int),
        "vba_export_step": ([v, v, v, v], C.c_int),
        "vba_export_reduced": ([v, v, C.c_double, v, v], C.c_int),
        "vba_apply_step": ([v, v], C.c_int),
        "vba_restore": ([v, v], C.c_int),
        "vba_accept": ([v, v], C.c_int),
        "vba_trial": ([v, v, C.c_double, C.c_int32, C.POINTER(VbaTrialResult)], C.c_int),
        "vba_solve": ([v, v, C.POINTER(VbaReport), C.POINTER(C.c_double), C.c_int32], C.c_int),
        "vba_download": ([v, v], C.c_int),
        "vba_launch_count": ([v], C.c_int64),
        "vba_stage_times": ([v, C.POINTER(C.c_double)], C.c_int),
        "vba_load_state": ([v, v], C.c_int),
        "vba_bind_inputs": ([v, v, v, v, C.c_int32], C.c_int),
        "vba_set_profiling": ([v, C.c_int32], C.c_int),
        "vba_stats": ([v, C.POINTER(C.c_int64)], C.c_int),
        "vba_gram_kind": ([v], C.c_int),
        "vba_chol_plan": ([C.c_int32, v, C.c_int32], C.c_int),
        "vba_copy_segments": ([v, C.c_int32, v], C.c_int),
        "vba_solve_times": ([v, C.POINTER(C.c_double)], C.c_int),
        "vba_spd_solve": ([v, C.c_int64, v, v, C.c_int32, v, C.POINTER(C.c_int32)], C.c_int),
        "vba_preintegrate": ([v, v, v, C.c_int64, v, C.c_int32, v, v, v, v, v], C.c_int),
        "vba_preint_scratch_bytes": ([C.c_int64], C.c_int64),
        "vba_preint_factor_records": ([v, v, C.c_int32, v, v], C.c_int),
        "vba_pg_create": ([C.POINTER(C.c_void_p), C.POINTER(VbaPgProblem), C.POINTER(VbaOptions), v], C.c_int),
        "vba_pg_destroy": ([v], C.c_int),
        "vba_pg_energy": ([v, v, C.POINTER(C.c_double)], C.c_int),
        "vba_pg_linearize": ([v, v], C.c_int),
        "vba_pg_export_normal_eq": ([v, v, v, v, v, v, v], C.c_int),
        "vba_pg_solve_step": ([v, v, C.c_double, C.c_int32], C.c_int),
        "vba_pg_export_step": ([v, v, v, v], C.c_int),
        "vba_pg_solve": ([v, v, C.POINTER(VbaReport), C.POINTER(C.c_double), C.c_int32], C.c_int),
        "vba_pg_download": ([v, v], C.c_int),
        "vba_init_inertial": ([C.POINTER(VbaInitProblem), C.POINTER(VbaInitOptions), v, C.POINTER(VbaInitResult),
                               C.POINTER(C.c_double), C.c_int32, v], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


_CUDA_OK = None


def cuda_available() -> bool:
    """torch.cuda.is_available(), evaluated once per process (each call of the torch
    function queries the driver: ~1 ms, the whole budget of a small window solve)."""
    global _CUDA_OK
    if _CUDA_OK is None:
        import torch
        _CUDA_OK = bool(torch.cuda.is_available())
    return _CUDA_OK


def check(rc: int):
    if rc != VBA_OK:
        msg = _lib.vba_last_error().decode() if _lib is not None else ""
        raise VbaError(rc, msg)


def spd_solve(H, b, mode: int = 0, iters: int = 0):
    """Solve H x = b for a dense SPD fp64 torch CUDA matrix (lower triangle used).

    mode 0: tcgen05 split-fp16 (3-product) Cholesky + fp64 iterative refinement (fp64 fallback
    on failed checks); mode 1: fp64 Cholesky (one CTA up to n = 232, else the DMMA tile DAG;
    VBA_CHOL=dag forces the DAG).  Returns (x, used_tensor_cores).
    Replaces np.linalg.solve(Hred, -gred) of solver.py:287.
    """
    import torch

    lib = load()
    n = H.shape[0]
    Hc = H.t().contiguous()          # column-major storage of H
    bc = b.contiguous()
    x = torch.empty_like(bc)
    info = (C.c_int32 * 2)(iters, 0)
    st = torch.cuda.current_stream(H.device).cuda_stream
    check(lib.vba_spd_solve(Hc.data_ptr(), n, bc.data_ptr(), x.data_ptr(), mode, st, info))
    return x, bool(info[0])
