"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module.  It is the checker the CUDA path is compared against, never the
thing that is measured as the product and never a fallback for it.

Two interchangeable CPU oracles live here:

* ``port``      -- oracle/tk_oracle.c, a C restatement of the reference's
                   compiled kernels (pkg/src/tenkern/_ckernels.pyx), loaded
                   through ctypes from oracle/libtk_oracle.so.
* ``reference`` -- the reference's own Cython kernel module, compiled from
                   /root/reference by ``make -C oracle ref`` into oracle/_ref/
                   (available wherever that build output exists, including the
                   GPU box, which receives the prebuilt .so).

The restatement is pinned against golden vectors that tests/golden/
make_golden.py produced by running the reference itself (tests/test_oracle.py).

Argument checks here mirror _check_ttv (pkg/src/tenkern/_ckernels.pyx:298-310)
and raise the same exception classes as the product package so parity tests can
compare error behaviour.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtk_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")

_lib = None


def build(quiet: bool = True) -> None:
    """Compile the C restatement (and the reference extension when /root/reference exists)."""
    targets = ["all"]
    if os.path.exists("/root/reference/pkg/src/tenkern/_ckernels.pyx"):
        targets.append("ref")
    subprocess.run(
        ["make", "-C", HERE, *targets, f"PY={sys.executable}"],
        check=True,
        stdout=subprocess.DEVNULL if quiet else None,
    )


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        c_dp = ctypes.POINTER(ctypes.c_double)
        c_ip = ctypes.POINTER(ctypes.c_int64)
        L.tko_dot.restype = ctypes.c_double
        L.tko_dot.argtypes = [c_dp, c_dp, ctypes.c_int64]
        L.tko_matvec.restype = None
        L.tko_matvec.argtypes = [c_dp, ctypes.c_int64, ctypes.c_int64, c_dp, c_dp]
        L.tko_ttv.restype = ctypes.c_int
        L.tko_ttv.argtypes = [ctypes.c_int32, c_ip, ctypes.c_int64, c_ip, c_dp, c_dp,
                              ctypes.c_int64, ctypes.c_int32, c_ip, c_dp, c_ip]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _errors():
    # Same classes the product raises, so tests compare types directly.
    from paper_2510_01495_b200 import errors
    return errors


def dot(x, y) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.shape[0] != y.shape[0]:
        raise _errors().DimensionError(
            f"dot: operand lengths differ: {x.shape[0]} vs {y.shape[0]}")
    return float(lib().tko_dot(_dp(x), _dp(y), x.shape[0]))


def matvec(a, x) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if a.shape[1] != x.shape[0]:
        raise _errors().DimensionError(
            f"matvec: matrix has {a.shape[1]} columns but vector has length {x.shape[0]}")
    y = np.empty(a.shape[0], dtype=np.float64)
    lib().tko_matvec(_dp(a), a.shape[0], a.shape[1], _dp(x), _dp(y))
    return y


def ttv_raw(subs, vals, shape, x, k):
    """Mode-k TTV over row-major (nnz, d) int64 subs; returns (subs, vals, shape)."""
    E = _errors()
    subs = np.ascontiguousarray(subs, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    shape = tuple(int(s) for s in shape)
    d, k = len(shape), int(k)
    if d < 2:
        raise E.OrderError(f"ttv: tensor order must be at least 2, got {d}")
    if k < 0 or k >= d:
        raise E.ModeError(f"ttv: mode {k} out of range for order-{d} tensor")
    if x.shape[0] != shape[k]:
        raise E.DimensionError(
            f"ttv: vector length {x.shape[0]} does not match shape[{k}] == {shape[k]}")
    new_shape = tuple(shape[m] for m in range(d) if m != k)
    nnz = subs.shape[0] if subs.ndim == 2 else 0
    out_subs = np.empty((max(nnz, 1), d - 1), dtype=np.int64)
    out_vals = np.empty(max(nnz, 1), dtype=np.float64)
    u = ctypes.c_int64(0)
    shp = np.asarray(shape, dtype=np.int64)
    rc = lib().tko_ttv(d, _ip(shp), nnz, _ip(subs), _dp(vals), _dp(x), x.shape[0], k,
                       _ip(out_subs), _dp(out_vals), ctypes.byref(u))
    if rc == 4:
        raise E.DimensionError(
            f"ttv: mode-{k} index out of range for a vector of length {x.shape[0]}")
    if rc != 0:
        raise MemoryError("oracle ttv: allocation failed")
    n = u.value
    return out_subs[:n].copy(), out_vals[:n].copy(), new_shape


def ttv_multi_dense(subs, vals, shape, vecs: dict, keep: int) -> np.ndarray:
    """Contract every mode but ``keep`` and return the dense order-1 result.

    The reference has no multi-vector TTV; following SURVEY.md
    §8c the oracle is chained single-mode ttv_raw in descending mode order (so
    the remaining mode numbers stay valid), then the order-1 triple is densified.
    """
    d = len(shape)
    cur_subs, cur_vals, cur_shape = np.asarray(subs), np.asarray(vals), tuple(shape)
    for m in sorted((m for m in range(d) if m != keep), reverse=True):
        cur_subs, cur_vals, cur_shape = ttv_raw(cur_subs, cur_vals, cur_shape, vecs[m], m)
    out = np.zeros(shape[keep], dtype=np.float64)
    out[cur_subs[:, 0]] = cur_vals
    return out


def mttkrp(subs, vals, shape, factors, n: int) -> np.ndarray:
    """MTTKRP oracle: column r is ttv_multi_dense with the vectors factors[m][:, r].

    The reference has no MTTKRP (the paper names it as future work);
    its definition here is the reference's own single-mode TTV chained per column
    (ttv_raw, which is pinned to the reference's goldens), SURVEY.md §8 f4.
    """
    d = len(shape)
    rank = next(np.asarray(f).shape[1] for m, f in enumerate(factors) if m != n)
    out = np.zeros((shape[n], rank), dtype=np.float64)
    for r in range(rank):
        vecs = {m: np.ascontiguousarray(np.asarray(factors[m], dtype=np.float64)[:, r])
                for m in range(d) if m != n}
        out[:, r] = ttv_multi_dense(subs, vals, shape, vecs, n)
    return out


def mttkrp_fused(subs, vals, shape, factors, n: int) -> np.ndarray:
    """Fused numpy restatement (row products, then a scatter-add) for larger cross-checks."""
    subs = np.asarray(subs)
    d = len(shape)
    w = np.asarray(vals, dtype=np.float64)[:, None]
    for m in range(d - 1, -1, -1):
        if m != n:
            w = w * np.asarray(factors[m], dtype=np.float64)[subs[:, m]]
    out = np.zeros((shape[n], w.shape[1]), dtype=np.float64)
    np.add.at(out, subs[:, n], w)
    return out


# -- the reference's own compiled module (oracle/_ref) ------------------------------------------

def reference_module():
    """Import the reference's compiled kernel module from oracle/_ref, or return None."""
    if not os.path.isdir(os.path.join(REF_DIR, "tenkern")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import tenkern._ckernels as ck  # noqa: WPS433 (reference build output)
    except ImportError:
        return None
    return ck
