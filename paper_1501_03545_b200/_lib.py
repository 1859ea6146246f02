"""ctypes binding of libhrgen_b200.so (include/hrgen_b200.h).

The product has exactly one compute path: this library on a CUDA device.
If the library is missing or no device is present, every entry point raises
NativeLibraryError -- nothing silently falls back to the CPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    InfeasibleParametersError,
    NativeLibraryError,
    OutOfBoundsError,
    ParameterDomainError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HRGEN_B200_LIB") or os.path.join(HERE, "libhrgen_b200.so")

HRG_OK = 0
HRG_ERR_PARAMETER_DOMAIN = 1
HRG_ERR_INFEASIBLE = 2
HRG_ERR_OUT_OF_BOUNDS = 3

ORDER_SAMPLE = 0
ORDER_ANGULAR = 1
MEM_HOST = 0
MEM_DEVICE = 1
TRIG_LIBM = 0   # glibc's sin/cos bit for bit (hrgen's arithmetic; the default)
TRIG_CR = 1     # correctly rounded sin/cos

# every symbol include/hrgen_b200.h declares, then include/hrgen_b200_debug.h's
# (checked against the headers by tests/test_abi.py)
EXPORTED = (
    "hrg_version", "hrg_last_error", "hrg_context_create", "hrg_context_destroy",
    "hrg_context_set_stream", "hrg_context_set_trig", "hrg_context_launches",
    "hrg_expected_avg_degree",
    "hrg_target_radius", "hrg_model_init", "hrg_generate", "hrg_sample_points",
    "hrg_edges_from_coords", "hrg_edges_brute_force", "hrg_result_sizes", "hrg_copy_result",
    "hrg_result_device_ptrs", "hrg_host_alloc", "hrg_host_free", "hrg_synchronize",
)
EXPORTED_DEBUG = ("hrg_debug_sincos", "hrg_debug_sincos_compare")


class Model(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("alpha", ctypes.c_double), ("R", ctypes.c_double),
        ("cosh_r_minus_1", ctypes.c_double), ("max_r", ctypes.c_double),
        ("rp_cap", ctypes.c_double), ("r_cap", ctypes.c_double),
        ("two_over_alpha", ctypes.c_double), ("sinh_half_alpha_r", ctypes.c_double),
    ]


class Shard(ctypes.Structure):
    _fields_ = [("index", ctypes.c_int32), ("count", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("m", ctypes.c_int64), ("nnz", ctypes.c_int64),
        ("candidates", ctypes.c_int64), ("radius", ctypes.c_double), ("alpha", ctypes.c_double),
        ("heavy_queries", ctypes.c_int64), ("heavy_chunks", ctypes.c_int64),
        ("t_sample_ms", ctypes.c_double), ("t_build_ms", ctypes.c_double),
        ("t_edges_ms", ctypes.c_double), ("t_sort_ms", ctypes.c_double),
        ("t_light_ms", ctypes.c_double), ("t_heavy_ms", ctypes.c_double),
        ("t_compact_ms", ctypes.c_double), ("t_rowsort_ms", ctypes.c_double),
        ("n_bands", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def _declare(L):
    S = ctypes.c_int
    sig = {
        "hrg_version": (ctypes.c_char_p, []),
        "hrg_last_error": (ctypes.c_char_p, []),
        "hrg_context_create": (S, [ctypes.c_int, _vp, ctypes.POINTER(_vp)]),
        "hrg_context_destroy": (S, [_vp]),
        "hrg_context_set_stream": (S, [_vp, _vp]),
        "hrg_context_set_trig": (S, [_vp, ctypes.c_int]),
        "hrg_context_launches": (S, [_vp, _i64p]),
        "hrg_expected_avg_degree": (S, [ctypes.c_int64, ctypes.c_double, ctypes.c_double, _dp]),
        "hrg_target_radius": (S, [ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_double, _dp]),
        "hrg_model_init": (S, [ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                               ctypes.POINTER(Model)]),
        "hrg_generate": (S, [_vp, ctypes.POINTER(Model), ctypes.c_uint64, ctypes.c_int,
                             ctypes.POINTER(Shard), ctypes.POINTER(Stats)]),
        "hrg_sample_points": (S, [_vp, ctypes.POINTER(Model), ctypes.c_uint64, ctypes.c_int,
                                  ctypes.c_int, _vp, _vp, _vp]),
        "hrg_edges_from_coords": (S, [_vp, ctypes.POINTER(Model), _vp, _vp, ctypes.c_int,
                                      ctypes.POINTER(Shard), ctypes.POINTER(Stats)]),
        "hrg_result_sizes": (S, [_vp, _i64p, _i64p]),
        "hrg_copy_result": (S, [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, ctypes.c_int]),
        "hrg_result_device_ptrs": (S, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                       ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                       ctypes.POINTER(_vp)]),
        "hrg_host_alloc": (S, [ctypes.c_size_t, ctypes.POINTER(_vp)]),
        "hrg_host_free": (S, [_vp]),
        "hrg_synchronize": (S, [_vp]),
        "hrg_debug_sincos": (S, [_vp, ctypes.c_int64, _vp, ctypes.c_int, _vp, _vp]),
        "hrg_debug_sincos_compare": (S, [_vp, ctypes.c_int64, ctypes.c_uint64, _vp, _vp]),
        "hrg_edges_brute_force": (S, [_vp, ctypes.c_int64, _vp, _vp, ctypes.c_int, ctypes.c_double,
                                      _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def load():
    """Load (never build) the library.  Raises NativeLibraryError if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (there is no CPU fallback)")
            try:
                L = ctypes.CDLL(LIB_PATH)
            except OSError as e:  # pragma: no cover
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
            _declare(L)
            _lib = L
    return _lib


def check(status):
    """Map a hrg_status to the reference's exception types."""
    if status == HRG_OK:
        return
    msg = load().hrg_last_error().decode(errors="replace")
    if status == HRG_ERR_PARAMETER_DOMAIN:
        raise ParameterDomainError(msg)
    if status == HRG_ERR_INFEASIBLE:
        raise InfeasibleParametersError(msg)
    if status == HRG_ERR_OUT_OF_BOUNDS:
        raise OutOfBoundsError(msg)
    raise NativeLibraryError(f"hrgen_b200 status {status}: {msg}")
