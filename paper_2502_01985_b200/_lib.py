"""ctypes binding of the C ABI in `include/fl_b200.h`.

The product path has exactly one implementation: the sm_100a kernels in
`_lib/libfl_b200.so`.  There is no CPU fallback -- if the library is missing
or no CUDA device is usable, every call raises `BackendUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FL_LIB_PATH") or os.path.join(HERE, "_lib", "libfl_b200.so")

FL_OK = 0
FL_ERR_SHAPE = 1
FL_ERR_OP = 2
FL_ERR_METADATA = 3
FL_ERR_CONFIG = 4
FL_ERR_DIVERGENCE = 5
FL_ERR_CUDA = 6
FL_ERR_ARG = 7

EW_IDS = {"scale": 0, "divide": 1, "square": 2, "abs": 3, "expm1": 4,
          "logistic_centered": 5}
MODEL_IDS = {"linreg": 0, "logreg": 1}


class BackendUnavailable(RuntimeError):
    """The B200 library could not be loaded or has no usable device."""


class FlError(RuntimeError):
    """CUDA / argument failure inside the library."""


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_PP = C.POINTER(C.c_void_p)

# name -> (argtypes); every function returns int status
SIGNATURES = {
    "fl_version": [],
    "fl_device_info": [C.c_int, C.POINTER(C.c_int), C.POINTER(_I64), C.POINTER(C.c_int),
                       C.POINTER(C.c_int)],
    "fl_table_create": [C.c_int, _I64, _I32, _PP],
    "fl_table_add_source": [_P, _I64, _I32, _P, _P, _P],
    "fl_table_finalize": [_P, _P],
    "fl_table_destroy": [_P],
    "fl_table_shape": [_P, C.POINTER(_I64), C.POINTER(_I32), C.POINTER(_I32)],
    "fl_table_layout": [_P, C.POINTER(_I32), C.POINTER(_I32), C.POINTER(_I32),
                        C.POINTER(_I32), C.POINTER(_I64)],
    "fl_table_gather_info": [_P, _I32, C.POINTER(_I32), C.POINTER(_I64), C.POINTER(_I32),
                             C.POINTER(_I32), C.POINTER(_I64)],
    "fl_table_selectors": [_P, _I32, _P, _P, _P, _P],
    "fl_table_perm": [_P, _P, _P],
    "fl_lmm": [_P, _P, _I32, _P, _P],
    "fl_tlmm": [_P, _P, _I32, _P, _P],
    "fl_rmm": [_P, _P, _I32, _P, _P],
    "fl_row_sum": [_P, _P, _P],
    "fl_col_sum": [_P, _P, _P],
    "fl_elementwise": [_P, _I32, _D, _PP, _P],
    "fl_materialize": [_P, _P, _P],
    "fl_crossprod": [_P, _P, _P],
    "fl_target_rows": [_P, _P, _I32, _P, _P],
    "fl_glm_create": [_P, _I32, _P, _D, _PP, _P],
    "fl_glm_partial": [_P, _P],
    "fl_glm_reduce_buffer": [_P, C.POINTER(C.c_void_p), C.POINTER(_I32)],
    "fl_glm_update": [_P, _P],
    "fl_glm_run": [_P, _I32, _P],
    "fl_glm_kernel_times": [_P, _I32, _P, _P],
    "fl_glm_result": [_P, _P, _P, _I32, C.POINTER(_I32), _P],
    "fl_glm_destroy": [_P],
    "fl_kmeans_create": [_P, _I32, _P, _PP, _P],
    "fl_kmeans_partial": [_P, _I32, _P],
    "fl_kmeans_reduce_buffer": [_P, C.POINTER(C.c_void_p), C.POINTER(_I32)],
    "fl_kmeans_update": [_P, _P],
    "fl_kmeans_run": [_P, _I32, _P],
    "fl_kmeans_kernel_times": [_P, _I32, _P, _P],
    "fl_kmeans_result": [_P, _P, _P, _P, _I32, C.POINTER(_I32), _P],
    "fl_kmeans_assignments64": [_P, _P, _P],
    "fl_kmeans_destroy": [_P],
    "fl_kmeans_path": [_P, C.POINTER(_I32)],
    "fl_glm_path": [_P, C.POINTER(_I32), C.POINTER(_D)],
    "fl_gnmf_create": [_P, _I32, _P, _P, _D, _PP, _P],
    "fl_gnmf_run": [_P, _I32, _P],
    "fl_gnmf_partial": [_P, _P],
    "fl_gnmf_kernel_times": [_P, _I32, _P, _P],
    "fl_gnmf_reduce_buffer": [_P, C.POINTER(C.c_void_p), C.POINTER(_I32)],
    "fl_gnmf_result": [_P, _P, _P, _P, _I32, C.POINTER(_I32), _P],
    "fl_gnmf_destroy": [_P],
    "fl_gnmf_path": [_P, C.POINTER(_I32)],
    "fl_comm_unique_id": [_P, _I32],
    "fl_comm_init": [_P, _I32, _I32, _I32, _I32, _PP],
    "fl_comm_allreduce": [_P, _P, C.c_int64, _P],
    "fl_comm_destroy": [_P],
    "fl_glm_set_comm": [_P, _P],
    "fl_kmeans_set_comm": [_P, _P],
    "fl_gnmf_set_comm": [_P, _P],
    "fl_tc_probe": [_I32, _P, _P, _P, _P, _I32, _I32, _P],
    "fl_tc_timing": [_I32, _I32, _I32, _I32, _I32, _I32, _I32, _P],
    "fl_tc_selftest": [_I32, _P, _P, _P, _I32, _I32, _P],
}

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return LIB_PATH


def load():
    """Load the CUDA library (once).  Raises BackendUnavailable if missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise BackendUnavailable(
                f"{LIB_PATH} is missing: build it with "
                "`python -m paper_2502_01985_b200._build` (there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib.fl_last_error.argtypes = []
        lib.fl_last_error.restype = C.c_char_p
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return sorted(list(SIGNATURES) + ["fl_last_error"])


def last_error() -> str:
    msg = load().fl_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = ""):
    """Map a status code to the reference's exception classes."""
    if status == FL_OK:
        return
    msg = last_error() or what
    if status == FL_ERR_SHAPE:
        from .sparse import ShapeError
        raise ShapeError(msg)
    if status == FL_ERR_OP:
        from .ops import OpError
        raise OpError(msg)
    if status == FL_ERR_METADATA:
        from .metadata import MetadataError, ValidationReport
        rep = ValidationReport()
        rep.add(None, "metadata", msg)
        raise MetadataError(rep)
    if status == FL_ERR_CONFIG:
        from .trainers import ConfigError
        raise ConfigError(msg)
    if status == FL_ERR_CUDA:
        raise BackendUnavailable(msg) if ("NoDevice" in msg or "InsufficientDriver" in msg
                                          or "no CUDA" in msg) else FlError(msg)
    raise FlError(f"{what}: {msg}")


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)


def device_info(device: int = 0) -> dict:
    sm = C.c_int()
    l2 = _I64()
    ma = C.c_int()
    mi = C.c_int()
    call("fl_device_info", device, C.byref(sm), C.byref(l2), C.byref(ma), C.byref(mi))
    return {"sm_count": sm.value, "l2_bytes": l2.value, "cc": (ma.value, mi.value)}
