"""The C-ABI library loads (no GPU needed) and matches include/vba.h."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "vba.h")
LIB = os.path.join(REPO, "paper_2512_02293_b200", "_vba.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", os.path.join(REPO, "paper_2512_02293_b200", "csrc"), "-j4"])
    return ctypes.CDLL(LIB)


def header_symbols():
    txt = open(HEADER).read()
    return re.findall(r"VBA_API[^;(]*?\b(vba_\w+)\s*\(", txt)


def test_header_declares_entry_points():
    names = header_symbols()
    for must in ("vba_create", "vba_solve", "vba_energy", "vba_linearize", "vba_solve_step",
                 "vba_apply_step", "vba_restore", "vba_set_collective", "vba_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_python_binding_covers_every_symbol():
    from paper_2512_02293_b200 import _lib
    assert set(header_symbols()) == set(_lib.EXPORTED)


def test_version_and_error_string_without_gpu(lib):
    lib.vba_version.restype = ctypes.c_int
    lib.vba_last_error.restype = ctypes.c_char_p
    assert lib.vba_version() == 1
    assert isinstance(lib.vba_last_error(), bytes)


def test_create_rejects_null_problem_without_touching_the_gpu(lib):
    ctx = ctypes.c_void_p()
    lib.vba_create.restype = ctypes.c_int
    assert lib.vba_create(ctypes.byref(ctx), None, None, None) == 1     # VBA_E_INVALID
    assert ctx.value is None


def _c_layout(struct, fields):
    src = ["#include <stdio.h>", "#include <stddef.h>", '#include "vba.h"', "int main(void){",
           f'printf("%zu\\n", sizeof({struct}));']
    src += [f'printf("%zu\\n", offsetof({struct}, {f}));' for f in fields]
    src += ["return 0;}"]
    d = os.path.join(REPO, "build")
    os.makedirs(d, exist_ok=True)
    c = os.path.join(d, f"layout_{struct}.c")
    exe = c[:-2]
    open(c, "w").write("\n".join(src))
    subprocess.check_call(["gcc", "-I", os.path.join(REPO, "include"), c, "-o", exe])
    out = subprocess.check_output([exe]).decode().split()
    return int(out[0]), [int(v) for v in out[1:]]


@pytest.mark.parametrize("cls,struct", [("VbaProblem", "vba_problem"), ("VbaOptions", "vba_options"),
                                        ("VbaReport", "vba_report"), ("VbaTrialResult", "vba_trial_result"),
                                        ("VbaPgProblem", "vba_pg_problem"), ("VbaInitProblem", "vba_init_problem"),
                                        ("VbaInitOptions", "vba_init_options"),
                                        ("VbaInitResult", "vba_init_result"), ("VbaCopySeg", "vba_copy_seg")])
def test_ctypes_struct_layout_matches_c(cls, struct):
    from paper_2512_02293_b200 import _lib
    S = getattr(_lib, cls)
    fields = [f[0] for f in S._fields_]
    size, offs = _c_layout(struct, fields)
    assert size == ctypes.sizeof(S)
    assert offs == [getattr(S, f).offset for f in fields]


def test_preintegration_entry_points_without_gpu(lib):
    """vba_preint_scratch_bytes / vba_preintegrate / vba_preint_factor_records validate their
    arguments on the host (VBA_E_INVALID) and accept empty windows without touching a GPU;
    the header's record sizes match the Python binding."""
    from paper_2512_02293_b200 import _lib
    L = _lib.load()
    hdr = open(os.path.join(REPO, "include", "vba.h")).read()
    assert f"#define VBA_PREINT_REC {_lib.PREINT_REC}" in hdr
    assert f"#define VBA_IMU_REC {_lib.IMU_REC}" in hdr
    assert L.vba_preint_scratch_bytes(-1) == -1
    assert L.vba_preint_scratch_bytes(1000) >= 1000 * 40 * 8
    assert L.vba_preintegrate(None, None, None, 0, None, 0, None, None, None, None, None) == 0     # empty
    assert L.vba_preintegrate(None, None, None, 0, None, -1, None, None, None, None, None) == 1    # invalid
    assert L.vba_preintegrate(None, None, None, 10, None, 2, None, None, None, None, None) == 1    # null buffers
    assert L.vba_preint_factor_records(None, None, 0, None, None) == 0
    assert L.vba_preint_factor_records(None, None, 3, None, None) == 1
    assert L.vba_copy_segments(None, 0, None) == 0      # nothing to copy: no device touched
    assert L.vba_copy_segments(None, 2, None) == 1      # null segment table
