"""ctypes binding of libtoepreg_b200.so (the C ABI in include/toepreg_b200.h).

There is no fallback: if the shared library or a CUDA device is missing,
every solve raises.  The library is built in-tree by ``make`` (or
``__graft_entry__.build()``) so the same ``.so`` travels to the GPU box.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtoepreg_b200.so")
# TR_LIB_PATH: load an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("TR_LIB_PATH", LIB_PATH)

VARIANTS = {"general": 0, "l2": 1, "gramian": 2}
FILLS = {"auto": 0, "zero": 1, "echo": 2}


class TrDesc(C.Structure):
    _fields_ = [
        ("variant", C.c_int32),
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("p_rows", C.c_int64),
        ("n_lim", C.c_int32),
        ("pivot_threshold", C.c_double),
        ("fill", C.c_int32),
        ("paired", C.c_int32),
        ("force_even", C.c_int32),
        ("refine", C.c_int32),
        ("refine_cg", C.c_int32),
        ("real_data", C.c_int32),
    ]


class TrDiag(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("difficult_points", C.c_int32),
        ("conditions_total", C.c_int64),
        ("recursion_depth", C.c_int32),
        ("retried_leaves", C.c_int32),
        ("max_column_scale", C.c_double),
        ("final_col_degrees", C.c_int64 * 8),
        ("relative_residual", C.c_double),
        ("trim_overflow", C.c_int32),
        ("refine_cg_iterations", C.c_int32),
        ("wall_time_s", C.c_double),
        ("rescued", C.c_int32),
    ]


# name -> (restype, argtypes); every symbol include/toepreg_b200.h declares
_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
SIGNATURES = {
    "tr_workspace_bytes": (C.c_size_t, [C.POINTER(TrDesc), _I64]),
    "tr_plan_info": (C.c_int, [C.POINTER(TrDesc), C.POINTER(_I64), C.POINTER(_I64),
                               C.POINTER(_I32), C.POINTER(_I64)]),
    "tr_solve_batch": (C.c_int, [C.POINTER(TrDesc), _I64, _P, _I64, _P, _I64, _P, _I64,
                                 _P, _I64, _P, _I64, _I32, _P, C.POINTER(TrDiag), _P,
                                 C.c_size_t, _P]),
    "tr_solve_batch_host": (C.c_int, [C.POINTER(TrDesc), _I64, _P, _I64, _P, _I64, _P, _I64,
                                      _P, _I64, _P, _I64, _I32, _P, C.POINTER(TrDiag)]),
    "tr_cg_workspace_bytes": (C.c_size_t, [C.POINTER(TrDesc), _I64]),
    "tr_cg_batch": (C.c_int, [C.POINTER(TrDesc), _I64, _P, _I64, _P, _I64, _P, _I64,
                              _P, _I64, _P, _I64, _I32, _I64, C.c_double, C.c_double,
                              _P, C.POINTER(_I64), _P, C.c_size_t, _P]),
    "tr_normal_apply": (C.c_int, [C.POINTER(TrDesc), _I64, _P, _I64, _P, _I64, _P, _I64,
                                  _P, _I64, _P, _P, _P, C.c_size_t, _P]),
    "tr_nudft": (C.c_int, [_P, _I64, _I64, _P, _I32, _I32, _P, _P]),
    "tr_fft": (C.c_int, [_P, _P, _I64, _I64, _I32, _P]),
    "tr_grid_eval": (C.c_int, [_P, _I64, _I64, _I64, _I64, _I64, _P, _P]),
    "tr_matpoly_mul": (C.c_int, [_P, _I64, _P, _I64, _I32, _P, _P]),
    "tr_assemble": (C.c_int, [C.POINTER(TrDesc), _P, _P, _P, _P, _P, _I32, _P, _P]),
    "tr_leaf": (C.c_int, [C.POINTER(TrDesc), _P, _I64, C.POINTER(_I64), _P, _I64,
                          C.POINTER(_I32), C.POINTER(C.c_double), C.POINTER(_I32), _P]),
    "tr_launch_count": (C.c_int64, []),
    "tr_kernel_timing": (C.c_int, [_I32]),
    "tr_kernel_stats": (C.c_int, [_I32, C.POINTER(C.c_double), C.POINTER(_I64)]),
    "tr_kernel_work_stats": (C.c_int, [_I32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "tr_fp64_peak": (C.c_int, [C.POINTER(C.c_double)]),
    "tr_fft_breakdown": (C.c_int, [C.POINTER(_I64), C.POINTER(C.c_double), C.c_int]),
    "tr_last_error": (C.c_char_p, []),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `make` or "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


KERNEL_CLASSES = ["assemble", "fft", "leaf_pivot", "leaf_build", "leaf_check", "leaf_exact",
                  "update", "combine", "normal", "finish"]


def kernel_stats():
    """{class: (total_ms, launches, alg_bytes, alg_flops)} since the last
    tr_kernel_timing call."""
    lib = load()
    out = {}
    for i, name in enumerate(KERNEL_CLASSES):
        ms, n = C.c_double(), C.c_int64()
        by, fl = C.c_double(), C.c_double()
        lib.tr_kernel_stats(i, C.byref(ms), C.byref(n))
        lib.tr_kernel_work_stats(i, C.byref(by), C.byref(fl))
        out[name] = (ms.value, n.value, by.value, fl.value)
    return out


def last_error() -> str:
    msg = load().tr_last_error()
    return msg.decode() if msg else ""
