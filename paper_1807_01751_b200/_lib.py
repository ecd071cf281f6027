"""ctypes binding of libbwm.so (the C ABI declared in include/bwm.h).

The library is built in-tree (``paper_1807_01751_b200/libbwm.so``, see build.py).  There
is deliberately no fallback: if the library or a CUDA device is missing, every entry
point raises.  Structs mirror include/bwm.h field for field.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libbwm.so"

BWM_OK = 0
BWM_E_NULL = -1
BWM_E_DIMS = -2
BWM_E_PARAMS = -3
BWM_E_SMEM = -4
BWM_E_DEVICE = -5
BWM_E_IO = -7
BWM_E_FORMAT = -8

BWM_NAN_FILL = 0
BWM_NAN_MASK = 1
NAN_MODES = {"fill": BWM_NAN_FILL, "mask": BWM_NAN_MASK}

INT64_MAX = (1 << 63) - 1
ABI_VERSION = 8


class Dims(C.Structure):
    _fields_ = [
        ("n_obs", C.c_int32),
        ("n_hist", C.c_int32),
        ("bandwidth", C.c_int32),
        ("n_params", C.c_int32),
        ("nan_mode", C.c_int32),
    ]


class Tables(C.Structure):
    _fields_ = [
        ("design", C.POINTER(C.c_double)),
        ("bound", C.POINTER(C.c_double)),
        ("trend_center", C.c_double),
        ("trend_scale", C.c_double),
    ]


class Outputs(C.Structure):
    _fields_ = [
        ("valid", C.c_void_p),
        ("first_idx", C.c_void_p),
        ("max_abs", C.c_void_p),
        ("beta", C.c_void_p),
        ("mo_mean", C.c_void_p),
        ("mosum", C.c_void_p),
        ("ld_out", C.c_int64),
        ("zero_sigma_pixel", C.c_void_p),
        ("first_break", C.c_void_p),
        ("max_abs_f64", C.c_void_p),
        ("detected", C.c_void_p),
        ("sup_stat", C.c_void_p),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("ring_mode", C.c_int32), ("ring_rows", C.c_int32), ("tmem_cols", C.c_int32), ("sms", C.c_int32),
        ("smem_tma", C.c_int64), ("smem_ldg", C.c_int64), ("ctas_per_sm_tma", C.c_int32),
        ("ctas_per_sm_ldg", C.c_int32), ("occupancy_tma", C.c_int32), ("force_ldg", C.c_int32),
        ("nan_mode", C.c_int32), ("masked_global", C.c_int32), ("ctas_per_sm_masked", C.c_int32),
        ("smem_masked", C.c_int64), ("const_bound", C.c_int32), ("ctas_per_sm_tma_lean", C.c_int32),
        ("precise", C.c_int32), ("mma", C.c_int32), ("smem_mma", C.c_int64), ("dyn_sched", C.c_int32), ("tall_stages", C.c_int32),
    ]


# (name, restype, argtypes) — every symbol include/bwm.h declares
SIGNATURES = [
    ("bwm_plan_create", C.c_int, [C.POINTER(Dims), C.POINTER(Tables), C.c_int, C.POINTER(C.c_void_p)]),
    ("bwm_plan_destroy", None, [C.c_void_p]),
    ("bwm_monitor", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.POINTER(Outputs), C.c_void_p]),
    ("bwm_monitor_host", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.POINTER(Outputs)]),
    ("bwm_monitor_file", C.c_int,
     [C.c_void_p, C.c_char_p, C.c_int64, C.c_int64, C.c_int, C.POINTER(Outputs)]),
    ("bwm_monitor_file_range", C.c_int,
     [C.c_void_p, C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.POINTER(Outputs)]),
    ("bwm_read_payload", C.c_int, [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int]),
    ("bwm_write_break_map", C.c_int64,
     [C.c_char_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    ("bwm_last_host_stats", C.c_int,
     [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("bwm_plan_info", C.c_int, [C.c_void_p, C.POINTER(PlanInfo)]),
    ("bwm_zero_sigma_init", C.c_int, [C.c_void_p, C.c_void_p]),
    ("bwm_null_draws", C.c_int,
     [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]),
    ("bwm_launch_count", C.c_int64, []),
    ("bwm_smem_bytes", C.c_int64, [C.POINTER(Dims)]),
    ("bwm_last_error", C.c_char_p, []),
    ("bwm_abi_version", C.c_int, []),
]

_lib = None


def load() -> C.CDLL:
    """Load libbwm.so (once).  Raises if it has not been built — no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("BWM_LIB", LIB_PATH))
    if not path.exists():
        raise RuntimeError(
            f"libbwm.so not found at {path}; build it with "
            "`python -m paper_1807_01751_b200.build` (there is no CPU fallback)"
        )
    lib = C.CDLL(str(path))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.bwm_abi_version() != ABI_VERSION:
        raise RuntimeError("libbwm ABI version mismatch; rebuild the library")
    _lib = lib
    return lib


def last_error() -> str:
    return load().bwm_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Map a libbwm return code onto the reference's exception types."""
    if rc == BWM_OK:
        return
    from .errors import DeviceError

    msg = f"{what}: {last_error()}"
    if rc in (BWM_E_DIMS, BWM_E_NULL, BWM_E_PARAMS):
        raise ValueError(msg)
    if rc == BWM_E_IO:
        raise OSError(msg)
    if rc == BWM_E_FORMAT:
        from .errors import StackFormatError

        raise StackFormatError(last_error())
    raise DeviceError(msg)


def launch_count() -> int:
    return int(load().bwm_launch_count())
