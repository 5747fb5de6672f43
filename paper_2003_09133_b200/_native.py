"""ctypes binding of the C-ABI library ``libhprime.so`` (include/lfbp_hprime.h).

The library is built in-tree by ``paper_2003_09133_b200.build`` (nvcc,
sm_100a).  There is no fallback: if the library is missing or a compute
entry point fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import DimsError, EvenPixelDims, FormatError, InvalidDims, IoError, LfbpError, NativeError

# LFBP_LIB_PATH: load another build of the library (same-box A/B of kernel versions)
LIB_PATH = os.environ.get("LFBP_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhprime.so")

(OK, ERR_INVALID_DIMS, ERR_EVEN_PIXEL_DIMS, ERR_CUDA, ERR_ARGUMENT, ERR_UNSUPPORTED, ERR_FORMAT, ERR_IO,
 ERR_DIMS) = range(9)
F32, F64 = 1, 2
HOST_REGISTER = 1
HOST_STAGE = 2

EXPORTS = (
    "lfbp_check_dims", "lfbp_dropped_source_count", "lfbp_hprime_device", "lfbp_hprime_host",
    "lfbp_hprime_multi", "lfbp_shard_planes", "lfbp_compare_device", "lfbp_plan_json",
    "lfbp_launch_count", "lfbp_last_error", "lfbp_version", "lfbp_plane_sums_device",
    "lfbp_lf5_read_header", "lfbp_lf5_create", "lfbp_lf5_transform_file", "lfbp_lf5_load_device",
    "lfbp_lf5_store_device", "lfbp_forward_project_device", "lfbp_backproject_device",
    "lfbp_safe_divide_device", "lfbp_forward_project2_device", "lfbp_max_device",
    "lfbp_safe_divide_peak_device", "lfbp_rl_update_device", "lfbp_host_alloc", "lfbp_host_free",
    "lfbp_host_cache_release", "lfbp_tune", "lfbp_plan_candidates", "lfbp_host_copy",
    "lfbp_synth_planes_device",
)

_lock = threading.Lock()
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_SIGS = {
    "lfbp_check_dims": (ctypes.c_int, [_i64p]),
    "lfbp_dropped_source_count": (ctypes.c_int64, [_i64p]),
    "lfbp_hprime_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64p, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]),
    "lfbp_hprime_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64p, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "lfbp_hprime_multi": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64p, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                         ctypes.c_int]),
    "lfbp_shard_planes": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int, _i64p, _i64p]),
    "lfbp_compare_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, _i64p,
                                           _i64p, ctypes.c_void_p]),
    "lfbp_plan_json": (ctypes.c_int, [_i64p, ctypes.c_int, ctypes.c_char_p, ctypes.c_int64]),
    "lfbp_plane_sums_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64p, ctypes.c_int,
                                              ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]),
    "lfbp_lf5_read_header": (ctypes.c_int, [ctypes.c_char_p, _i64p, ctypes.POINTER(ctypes.c_int)]),
    "lfbp_lf5_create": (ctypes.c_int, [ctypes.c_char_p, _i64p, ctypes.c_int]),
    "lfbp_lf5_transform_file": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int]),
    "lfbp_lf5_load_device": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_void_p]),
    "lfbp_lf5_store_device": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_void_p]),
    "lfbp_forward_project_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _i64p, ctypes.c_void_p,
                                                   ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "lfbp_forward_project2_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, _i64p,
                                                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                                    ctypes.c_void_p]),
    "lfbp_backproject_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _i64p, ctypes.c_int, ctypes.c_void_p,
                                               ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "lfbp_safe_divide_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
    "lfbp_max_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "lfbp_safe_divide_peak_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                    ctypes.c_int64, ctypes.c_double, ctypes.c_void_p,
                                                    ctypes.c_void_p]),
    "lfbp_rl_update_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
    "lfbp_host_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "lfbp_host_free": (ctypes.c_int, [ctypes.c_void_p]),
    "lfbp_host_cache_release": (ctypes.c_int, []),
    "lfbp_tune": (ctypes.c_int, [_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int64]),
    "lfbp_plan_candidates": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.c_int]),
    "lfbp_host_copy": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]),
    "lfbp_synth_planes_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _i64p, ctypes.c_int64,
                                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.c_void_p]),
    "lfbp_launch_count": (ctypes.c_int64, []),
    "lfbp_last_error": (ctypes.c_char_p, []),
    "lfbp_version": (ctypes.c_char_p, []),
}


def lib():
    """The loaded library; raises ``NativeError`` if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (there is no CPU fallback)")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def dims_array(shape) -> ctypes.Array:
    return (ctypes.c_int64 * 5)(*[int(v) for v in shape])


def last_error() -> str:
    return lib().lfbp_last_error().decode(errors="replace")


def check(rc: int, invalid=InvalidDims, even=EvenPixelDims) -> None:
    """Map a status code onto the reference's exception types."""
    if rc == OK:
        return
    msg = last_error()
    if rc == ERR_INVALID_DIMS:
        raise invalid(msg)
    if rc == ERR_EVEN_PIXEL_DIMS:
        raise even(msg)
    if rc == ERR_CUDA:
        raise NativeError(msg)
    if rc == ERR_FORMAT:
        raise FormatError(msg)
    if rc == ERR_IO:
        raise IoError(msg)
    if rc == ERR_DIMS:
        raise DimsError(msg)
    if rc in (ERR_ARGUMENT, ERR_UNSUPPORTED):
        raise LfbpError(msg) if rc == ERR_UNSUPPORTED else ValueError(msg)
    raise NativeError(f"status {rc}: {msg}")


def launch_count() -> int:
    return int(lib().lfbp_launch_count())
