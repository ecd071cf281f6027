"""The C-ABI boundary (include/bwm.h) without a GPU: libbwm.so loads, exports every
declared entry point, reports its ABI version and validates dimensions."""

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "bwm.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(bwm_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_hot_call():
    names = declared_functions()
    for required in ("bwm_plan_create", "bwm_monitor", "bwm_monitor_host", "bwm_plan_destroy", "bwm_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1807_01751_b200 import _lib

    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(bwm_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, f"declared in bwm.h but not exported: {missing}"
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_functions()) <= bound, "every ABI function needs a ctypes signature"
    for name in declared_functions():
        assert hasattr(lib, name)


def test_abi_version_and_error_string():
    from paper_1807_01751_b200 import _lib

    lib = _lib.load()
    assert lib.bwm_abi_version() == _lib.ABI_VERSION == 8
    assert isinstance(lib.bwm_last_error(), bytes)


@pytest.mark.parametrize(
    "dims,code",
    [
        ((228, 114, 28, 8), None),          # C1-C3 geometry
        ((1000, 500, 250, 14), None),       # C4
        ((228, 228, 28, 8), -2),            # n >= N
        ((228, 114, 0, 8), -2),             # h < 1
        ((228, 114, 115, 8), -2),           # h > n
        ((228, 8, 4, 8), -2),               # n <= p
        ((228, 114, 28, 7), -3),            # odd parameter count
        ((228, 114, 28, 20), -3),           # k > 8
        ((228, 114, 28, 8, 1), None),       # masked-NaN mode, tables in shared memory
        ((1000, 500, 250, 14, 1), None),    # masked-NaN mode, x x^T table + rings in global memory
        ((228, 114, 28, 8, 2), -3),         # unknown nan_mode
    ],
)
def test_dimension_validation(dims, code):
    from paper_1807_01751_b200 import _lib

    lib = _lib.load()
    d = _lib.Dims(*dims)
    r = lib.bwm_smem_bytes(C.byref(d))
    if code is None:
        assert r > 0 and r <= 227 * 1024
    else:
        assert r == code
        assert lib.bwm_last_error()


def test_null_arguments_rejected_without_device():
    from paper_1807_01751_b200 import _lib

    lib = _lib.load()
    assert lib.bwm_monitor(None, None, 0, 0, 0, None, None) == _lib.BWM_E_NULL
    assert lib.bwm_monitor_host(None, None, 0, 0, 0, None) == _lib.BWM_E_NULL
    plan = C.c_void_p()
    assert lib.bwm_plan_create(None, None, 0, C.byref(plan)) == _lib.BWM_E_NULL
    assert lib.bwm_plan_info(None, None) == _lib.BWM_E_NULL


def test_sass_contains_blackwell_async_copy_and_tensor_memory():
    """The default kernel is built for sm_100a and uses tensor TMA (UTMALDG) and Tensor
    Memory (LDTM/STTM) — evidence checked on the shipped .so, not on a cached build."""
    from paper_1807_01751_b200 import _lib

    out = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(_lib.LIB_PATH)], capture_output=True,
                                       text=True).stdout
    for mnemonic in ("UTMALDG", "LDTM", "STTM", "FFMA2", "SYNCS"):
        assert mnemonic in out, mnemonic


@pytest.mark.gpu
def test_plan_requires_intercept_design_row():
    """bwm_tables documents design row 0 as the intercept (1 at every date): the window-sum
    formulation folds that row's window sum into a constant, so a plan with another row 0 is
    refused (BWM_E_DIMS) rather than computed wrongly."""
    import numpy as np

    from paper_1807_01751_b200 import _lib

    lib = _lib.load()
    N, n, h, p = 60, 30, 10, 4
    t = np.arange(1.0, N + 1)
    design = np.ascontiguousarray(np.stack([np.ones(N), (t - 15.5) / 14.5, np.sin(t / 3), np.cos(t / 3)]))
    bound = np.full(N - n, 3.0)
    dbl = C.POINTER(C.c_double)
    dims = _lib.Dims(N, n, h, p, 0)
    plan = C.c_void_p()
    ok = _lib.Tables(design.ctypes.data_as(dbl), bound.ctypes.data_as(dbl), 15.5, 14.5)
    assert lib.bwm_plan_create(C.byref(dims), C.byref(ok), 0, C.byref(plan)) == 0
    lib.bwm_plan_destroy(plan)
    bad = design.copy()
    bad[0, 7] = 2.0
    tb = _lib.Tables(bad.ctypes.data_as(dbl), bound.ctypes.data_as(dbl), 15.5, 14.5)
    plan = C.c_void_p()
    assert lib.bwm_plan_create(C.byref(dims), C.byref(tb), 0, C.byref(plan)) == -2
    assert b"intercept" in lib.bwm_last_error()
