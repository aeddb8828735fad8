"""ctypes binding of libtk_b200.so (the C ABI in include/tk_b200.h).

This is the only module that touches the shared library.  There is no fallback: if the
library is missing, importing a kernel raises, and on a machine without a GPU every
compute entry point raises DeviceError from the CUDA runtime's own message.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtk_b200.so")

TK_OK, TK_EDIM, TK_EMODE, TK_EORDER, TK_EINDEX, TK_ECUDA, TK_ENCCL, TK_EARG, TK_ENOMEM = 0, 1, 2, 3, 4, 6, 7, 8, 9
MAX_ORDER = 16

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); every symbol include/tk_b200.h declares
SIGNATURES = {
    "tk_last_error": (ctypes.c_char_p, []),
    "tk_version": (ctypes.c_int, []),
    "tk_last_call_seconds": (ctypes.c_double, []),
    "tk_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "tk_dot_f64_device": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, _vp]),
    "tk_dot_f64_host": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _c_dp]),
    "tk_matvec_f64_device": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp]),
    "tk_matvec_f64_host": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp]),
    "tk_ttv_f64_device": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int64, _vp, _vp, _vp, _vp,
                                         ctypes.c_int64, ctypes.c_int32, _vp, _vp, _c_i64p, _vp]),
    "tk_ttv_f64_host": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int64, _vp, _vp, _vp,
                                       ctypes.c_int64, ctypes.c_int32, _vp, _vp, _c_i64p]),
    "tk_group_sum_f64_host": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp, _vp, _c_i64p]),
    "tk_ttv_dense_f64_device": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int64, _vp, _vp, _vp,
                                               ctypes.c_int32, _vp, _vp, _vp]),
    "tk_ttv_dense_f64_device_peers": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int64, _vp, _vp,
                                                     ctypes.c_int32, _vp, _vp, ctypes.c_int32, ctypes.c_int64,
                                                     ctypes.c_int64, _vp]),
    "tk_ipc_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "tk_ipc_free": (ctypes.c_int, [_vp]),
    "tk_ipc_get_handle": (ctypes.c_int, [_vp, _vp]),
    "tk_ipc_open": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_void_p)]),
    "tk_ipc_close": (ctypes.c_int, [_vp]),
    "tk_mttkrp_f64_device": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int64, _vp, _vp, _vp,
                                            ctypes.c_int32, ctypes.c_int64, _vp, _vp, _vp]),
    "tk_mttkrp_f64_host": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int64, _vp, _vp,
                                          ctypes.c_int32, ctypes.c_int64, _vp, _vp]),
    "tk_gen_coo_device": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int64, ctypes.c_double,
                                         ctypes.c_int32, ctypes.c_uint64, _vp, _vp, _vp]),
    "tk_gen_uniform_device": (ctypes.c_int, [ctypes.c_int64, ctypes.c_uint64, _vp, _vp]),
    "tk_ttv_workspace": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                        ctypes.POINTER(ctypes.c_size_t)]),
    "tk_dot_f64_device_timed": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, _vp, ctypes.POINTER(ctypes.c_float)]),
    "tk_matvec_f64_device_timed": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp,
                                                  ctypes.POINTER(ctypes.c_float)]),
    "tk_ttv_f64_device_timed": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int64, _vp, _vp, _vp, _vp,
                                               ctypes.c_int64, ctypes.c_int32, _vp, _vp, _c_i64p, _vp,
                                               ctypes.POINTER(ctypes.c_float)]),
    "tk_multi_init": (ctypes.c_int, [ctypes.c_int32, _vp]),
    "tk_multi_ttv_f64": (ctypes.c_int, [ctypes.c_int32, _c_i64p, ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp,
                                        _vp, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp]),
    "tk_multi_free": (ctypes.c_int, []),
    "tk_nccl_load": (ctypes.c_int, [ctypes.c_char_p]),
    "tk_nccl_version": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "tk_nccl_get_unique_id": (ctypes.c_int, [_vp]),
    "tk_nccl_comm_init": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "tk_nccl_comm_free": (ctypes.c_int, [_vp]),
    "tk_nccl_rank": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
    "tk_nccl_counts_start": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, ctypes.POINTER(ctypes.c_int32)]),
    "tk_nccl_counts_wait": (ctypes.c_int, [_vp, ctypes.c_int32, _c_i64p]),
    "tk_nccl_gather_rows": (ctypes.c_int, [_vp, ctypes.c_int32, _vp, _vp, ctypes.c_int32, _c_i64p, _vp, _vp, _vp]),
    "tk_nccl_allgather_bytes": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64]),
    "tk_nccl_barrier": (ctypes.c_int, [_vp, _vp]),
    "tk_nccl_allreduce_sum_f64": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp]),
    "tk_read_floor_f64_device": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp]),
    "tk_timer_start": (ctypes.c_int, [_vp]),
    "tk_timer_stop": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_float)]),
    "tk_release": (ctypes.c_int, []),
    "tk_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "tk_host_free": (ctypes.c_int, [_vp]),
    "tk_last_kernel_ms": (ctypes.c_double, []),
    "tk_launch_count": (ctypes.c_longlong, []),
}

_lib = None


def load():
    """Load (once) and return the library; raises ImportError if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2510_01495_b200/csrc` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_STATUS_EXC = {
    TK_EDIM: errors.DimensionError,
    TK_EINDEX: errors.DimensionError,
    TK_EMODE: errors.ModeError,
    TK_EORDER: errors.OrderError,
    TK_EARG: errors.ConfigError,
    TK_ECUDA: errors.DeviceError,
    TK_ENCCL: errors.DeviceError,
    TK_ENOMEM: errors.DeviceError,
}


def check(rc: int) -> None:
    if rc != TK_OK:
        msg = load().tk_last_error().decode(errors="replace")
        raise _STATUS_EXC.get(rc, errors.DeviceError)(msg)


def i64_array(values):
    arr = (ctypes.c_int64 * len(values))(*[int(v) for v in values])
    return arr


def ptr_array(ptrs):
    return (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])


def device_count() -> int:
    n = ctypes.c_int(0)
    load().tk_device_count(ctypes.byref(n))
    return n.value
