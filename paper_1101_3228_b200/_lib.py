"""ctypes binding of include/qtree_cuda.h (libqtree_cuda.so, built in-tree).

There is deliberately no fallback: if the CUDA library is missing or cannot be
loaded, importing the estimator API raises. The library itself refuses to run
without a CUDA device (QT_ERR_DEVICE).
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

QT_OK, QT_ERR_INVALID_ARGUMENT, QT_ERR_CONFIG, QT_ERR_IO, QT_ERR_NUMERIC, QT_ERR_DEVICE = range(6)


class QtChain(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layers", C.c_int32),
                ("step", C.POINTER(C.c_double)), ("marginal", C.POINTER(C.c_double))]


class QtGrids(C.Structure):
    _fields_ = [("dim", C.c_int32), ("layers", C.c_int32),
                ("sizes", C.POINTER(C.c_uint64)), ("points", C.POINTER(C.c_double))]


class QtModelParams(C.Structure):
    _fields_ = [("s0", C.c_double), ("sigma1", C.c_double), ("sigma2", C.c_double),
                ("alpha1", C.c_double), ("alpha2", C.c_double), ("rho", C.c_double),
                ("r", C.c_double), ("strike", C.c_double), ("horizon", C.c_double),
                ("steps", C.c_int32), ("gbm_rho", C.c_double * 3)]


_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)

_SIGS = {
    "qt_chain_coefficients": [C.c_int32, C.POINTER(QtModelParams), _f64p, _f64p],
    "qt_estimate": [C.c_int32, C.POINTER(QtChain), C.POINTER(QtGrids), C.c_uint64, C.c_int32,
                    C.c_uint64, C.c_int32, _u64p, _u64p, _f64p, _f64p],
    "qt_estimate_device": [C.c_int32, C.POINTER(QtChain), C.POINTER(QtGrids), C.c_uint64,
                           C.c_int32, C.c_uint64, C.c_int32, C.POINTER(C.c_void_p), _f64p],
    "qt_dtree_destroy": [C.c_void_p],
    "qt_dtree_info": [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                      C.POINTER(C.c_uint64), _u64p, C.c_uint64, C.POINTER(C.c_int32)],
    "qt_dtree_device_arrays": [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                               C.POINTER(C.c_void_p)],
    "qt_dtree_download": [C.c_void_p, _u64p, _u64p, _f64p],
    "qt_dtree_stopping": [C.c_void_p, _f64p, _f64p, _u8p, _f64p],
    "qt_dtree_swing": [C.c_void_p, _f64p, C.c_int32, C.c_int32, _f64p, _f64p, _u8p],
    "qt_estimate_normals": [C.c_int32, C.POINTER(QtChain), C.POINTER(QtGrids), C.c_uint64,
                            _f64p, _u64p, _u64p, _f64p],
    "qt_accumulate_paths": [C.POINTER(QtChain), C.POINTER(QtGrids), C.c_int32, C.c_uint64,
                            C.c_uint64, C.c_uint64, C.c_uint64, _u64p, _u64p],
    "qt_plan_create": [C.POINTER(QtChain), C.POINTER(QtGrids), C.c_int32, C.POINTER(C.c_void_p)],
    "qt_plan_destroy": [C.c_void_p],
    "qt_plan_layout": [C.c_void_p, _u64p, _u64p],
    "qt_plan_count": [C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64,
                      C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)],
    "qt_plan_finalize": [C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                         C.c_void_p, C.POINTER(C.c_int32)],
    "qt_nearest": [C.c_int32, C.c_uint64, _f64p, C.c_uint64, _f64p, _u64p],
    "qt_bdp_stopping": [C.c_int32, _u64p, _u64p, _f64p, _f64p, _f64p, _u8p, _f64p],
    "qt_bdp_swing": [C.c_int32, _u64p, _u64p, _f64p, _f64p, C.c_int32, C.c_int32, _f64p, _f64p,
                     _u8p],
    "qt_bdp_cond_expectation": [C.c_uint64, C.c_uint64, _u64p, _f64p, _f64p, _f64p],
    "qt_path_normals": [C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _f64p],
    "qt_uniforms": [C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, _f64p],
    "qt_set_fast_path": [C.c_int32],
    "qt_fast_stats": [_u64p],
    "qt_plan_fast_stats": [C.c_void_p, _u64p],
    "qt_fast_bounds_check": [_f64p],
    "qt_math_checksum": [C.c_int32, _u64p],
    "qt_apx_bounds_check": [_f64p],
    "qt_lloyd_build_stream": [C.c_int32, C.c_uint64, C.c_int32, C.c_uint64, _u64p,
                              C.POINTER(C.c_int32), _f64p, _f64p, _f64p],
    "qt_distortion_stream": [C.c_int32, C.c_uint64, _f64p, C.c_uint64, _u64p,
                             C.POINTER(C.c_int32), _f64p, _f64p, _f64p],
    "qt_lloyd_iterate": [C.c_int32, C.c_uint64, _f64p, C.c_uint64, _f64p, _f64p],
    "qt_distortion_points": [C.c_int32, C.c_uint64, _f64p, C.c_uint64, _f64p, _f64p, _f64p],
    "qt_plan_cache_clear": [],
    "qt_payoff_table": [C.c_int32, C.c_int32, C.POINTER(QtModelParams), _f64p, C.c_int32, _u64p,
                        _f64p, _f64p],
    "qt_lloyd_build": [C.c_int32, C.c_uint64, C.c_int32, C.c_uint64, C.c_uint64, _f64p, C.c_uint64,
                       _f64p, _f64p],
    "qt_bench_pi": [C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, _u64p, _f64p,
                    _f64p, _f64p],
    "qt_bench_nn": [C.c_uint64, C.c_uint64, C.c_uint64, _u64p, _f64p],
    "qt_save_tree": [C.c_char_p, C.c_int32, C.c_int32, _u64p, _f64p, C.c_uint64, C.c_void_p,
                     C.c_void_p, C.c_void_p, C.c_int32],
    "qt_tree_file_info": [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                          C.POINTER(C.c_uint64), _u64p, C.c_uint64],
    "qt_load_tree": [C.c_char_p, C.c_int32, C.c_int32, _u64p, _f64p, _u64p, C.c_uint64, _u64p,
                     _f64p, C.c_uint64],
    "qt_save_grid": [C.c_char_p, C.c_int32, C.c_uint64, _f64p],
    "qt_load_grid": [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_uint64), _f64p, C.c_uint64],
}

# Every symbol include/qtree_cuda.h declares (checked by tests/test_boundary.py).
EXPORTS = sorted(list(_SIGS) + ["qt_last_error", "qt_version", "qt_kernel_launches"])

_lib = None


def lib():
    """Load libqtree_cuda.so (once). Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(
                f"{LIB} is missing: build it with `python -m paper_1101_3228_b200.build` "
                "(there is no CPU fallback for the estimator)")
        L = C.CDLL(LIB)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.qt_last_error.restype = C.c_char_p
        L.qt_version.restype = C.c_char_p
        L.qt_kernel_launches.restype = C.c_uint64
        _lib = L
    return _lib


def last_error() -> str:
    return lib().qt_last_error().decode()
