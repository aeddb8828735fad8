"""The B200 kernel module: the drop-in replacement for the reference's compiled kernels.

Satisfies the reference's kernel-module protocol (pkg/src/tenkern/backend.py:33-49 hands
out a module with ``BACKEND``, ``SELF_TIMED``, ``dot``, ``matvec``, ``ttv_raw`` and the
``*_timed`` entry points of pkg/src/tenkern/_ckernels.pyx:76-122, 370-388), so it plugs into
``tenhost.BoundKernelSet(kernel_module=...)`` (pkg/hostbench/src/tenhost/bindings.py:50-54),
which passes ``release_gil`` positionally, and into the reference's benchmark registry
(``ImplEntry``, pkg/src/tenkern/bench.py:191-215; see ``registry.py``).

Every call crosses the C ABI of libtk_b200.so with host buffers (``tk_*_host``): operands are
copied to HBM, the sm_100a kernels run, the result is copied back.  ctypes releases the GIL
for the duration of the foreign call regardless of ``release_gil``; results are identical
either way (the reference's contract, test_backend.py:64-78).

Device-resident data (no host copies) goes through :mod:`paper_2510_01495_b200.device`.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DimensionError, ModeError, OrderError

BACKEND = "b200"
SELF_TIMED = True

_i64p = ctypes.POINTER(ctypes.c_int64)


def _f64(a, ndim):
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.ndim != ndim:
        raise DimensionError(f"expected a {ndim}-D float64 array, got ndim={arr.ndim}")
    return arr


class _PinnedBlock:
    """A cached pinned result block (tk_host_alloc); numpy views keep it alive, and it goes back
    to the library's cache when the last view is dropped."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr = ptr
        self.__array_interface__ = {"data": (ptr, False), "shape": (nbytes,), "typestr": "|u1", "version": 3}

    def __del__(self):
        try:
            _lib.load().tk_host_free(self.ptr)
        except Exception:  # interpreter shutdown
            pass


_POOLED_RESULT_BYTES = 64 << 20


def _result_arrays(rows: int, cols: int):
    """(subs[rows, cols] int64, vals[rows] float64) for a host-call result.  Large results come
    from the library's pinned cache, so the device writes them directly; small ones (and any
    request past the cache cap) are ordinary owned arrays."""
    nbytes = rows * (cols + 1) * 8
    if nbytes >= _POOLED_RESULT_BYTES:
        p = ctypes.c_void_p()
        _lib.check(_lib.load().tk_host_alloc(nbytes, ctypes.byref(p)))
        if p.value:
            buf = np.asarray(_PinnedBlock(p.value, nbytes))
            cut = rows * cols * 8
            return buf[:cut].view(np.int64).reshape(rows, cols), buf[cut:].view(np.float64), True
    return np.empty((rows, cols), dtype=np.int64), np.empty(rows, dtype=np.float64), False


def _check_dot(x, y):
    if x.shape[0] != y.shape[0]:
        raise DimensionError(f"dot: operand lengths differ: {x.shape[0]} vs {y.shape[0]}")


def _check_matvec(a, x):
    if a.shape[1] != x.shape[0]:
        raise DimensionError(
            f"matvec: matrix has {a.shape[1]} columns but vector has length {x.shape[0]}")


def _dot(x, y) -> float:
    # structural guard (memory safety) is always on, like the Cython memoryview shapes
    _check_dot(x, y)
    out = ctypes.c_double(0.0)
    _lib.check(_lib.load().tk_dot_f64_host(x.ctypes.data, y.ctypes.data, x.shape[0], ctypes.byref(out)))
    return float(out.value)


def _matvec(a, x) -> np.ndarray:
    _check_matvec(a, x)
    y = np.empty(a.shape[0], dtype=np.float64)
    _lib.check(_lib.load().tk_matvec_f64_host(a.ctypes.data, a.shape[0], a.shape[1], x.ctypes.data, y.ctypes.data))
    return y


def dot(x, y, release_gil=False) -> float:
    """Replaces _ckernels.dot (pyx:76-83)."""
    return _dot(_f64(x, 1), _f64(y, 1))


def matvec(a, x, release_gil=False) -> np.ndarray:
    """Replaces _ckernels.matvec (pyx:86-95); returns a fresh float64 vector."""
    return _matvec(_f64(a, 2), _f64(x, 1))


def _ttv_host(subs, vals, shape, x, k):
    shape = tuple(int(s) for s in shape)
    d = len(shape)
    k = int(k)
    # structural guards, always on (_check_ttv, pyx:298-310)
    if d < 2:
        raise OrderError(f"ttv: tensor order must be at least 2, got {d}")
    if k < 0 or k >= d:
        raise ModeError(f"ttv: mode {k} out of range for order-{d} tensor")
    xv = _f64(x, 1)
    if xv.shape[0] != shape[k]:
        raise DimensionError(
            f"ttv: vector length {xv.shape[0]} does not match shape[{k}] == {shape[k]}")
    sv = np.ascontiguousarray(subs, dtype=np.int64)
    if sv.size == 0:
        sv = sv.reshape(0, d)
    vv = _f64(vals, 1)
    if sv.ndim != 2 or sv.shape[1] != d or sv.shape[0] != vv.shape[0]:
        raise DimensionError(f"ttv: subs of shape {sv.shape} and {vv.shape[0]} values do not match order {d}")
    nnz = sv.shape[0]
    new_shape = tuple(shape[m] for m in range(d) if m != k)
    out_subs, out_vals, pooled = _result_arrays(max(nnz, 1), d - 1)
    u = ctypes.c_int64(0)
    shp = _lib.i64_array(shape)
    _lib.check(_lib.load().tk_ttv_f64_host(d, shp, nnz, sv.ctypes.data, vv.ctypes.data, xv.ctypes.data,
                                            xv.shape[0], k, out_subs.ctypes.data, out_vals.ctypes.data,
                                            ctypes.byref(u)))
    n = u.value
    if pooled:  # exact-size views of the cached pinned block (released when the caller drops them)
        return out_subs[:n], out_vals[:n], new_shape
    # fresh, owned, exact-size outputs like the reference's copy-out (pyx:367), without a second
    # host copy: the capacity-sized buffers are shrunk in place (realloc; pages past u were never
    # touched, so they were never committed)
    out_subs.resize((n, d - 1), refcheck=False)
    out_vals.resize((n,), refcheck=False)
    return out_subs, out_vals, new_shape


def ttv_raw(subs, vals, shape, x, k, release_gil=False):
    """Mode-k TTV over raw COO buffers -> (new_subs, new_vals, new_shape).

    Replaces _ckernels.ttv_raw (pyx:370-374): bit-identical coordinates and values.
    """
    return _ttv_host(subs, vals, shape, x, k)


def _native_seconds() -> float:
    return float(_lib.load().tk_last_call_seconds())


def dot_timed(x, y, checked=False):
    """(value, elapsed_s) with elapsed measured on the native side (pyx:98-107)."""
    xv, yv = _f64(x, 1), _f64(y, 1)
    value = _dot(xv, yv)
    return value, _native_seconds()


def matvec_timed(a, x, checked=False):
    """(out, elapsed_s), output allocation included as in the reference (pyx:110-122)."""
    av, xv = _f64(a, 2), _f64(x, 1)
    out = _matvec(av, xv)
    return out, _native_seconds()


def ttv_timed(subs, vals, shape, x, k):
    """((new_subs, new_vals, new_shape), elapsed_s) (pyx:377-388)."""
    res = _ttv_host(subs, vals, shape, x, k)
    return res, _native_seconds()
