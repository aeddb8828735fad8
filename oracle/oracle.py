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


# -- host twin of the device generator (oracle/tk_gen_host.cpp) ---------------------------------

GEN_LIB_PATH = os.path.join(HERE, "libtk_gen_host.so")
_gen = None


def gen_lib():
    global _gen
    if _gen is None:
        if not os.path.exists(GEN_LIB_PATH):
            build()
        L = ctypes.CDLL(GEN_LIB_PATH)
        c_dp = ctypes.POINTER(ctypes.c_double)
        c_ip = ctypes.POINTER(ctypes.c_int64)
        L.tkg_gen_coo.restype = ctypes.c_int
        L.tkg_gen_coo.argtypes = [ctypes.c_int, c_ip, ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                  ctypes.c_uint64, ctypes.c_int, c_ip, c_dp]
        L.tkg_gen_uniform.restype = None
        L.tkg_gen_uniform.argtypes = [ctypes.c_int64, ctypes.c_uint64, c_dp]
        L.tkg_zipf_cdf.restype = None
        L.tkg_zipf_cdf.argtypes = [ctypes.c_int64, ctypes.c_double, c_dp]
        L.tkg_ln.restype = ctypes.c_double
        L.tkg_ln.argtypes = [ctypes.c_double]
        L.tkg_cos2pi.restype = ctypes.c_double
        L.tkg_cos2pi.argtypes = [ctypes.c_double]
        L.tkg_shard_bounds.restype = None
        L.tkg_shard_bounds.argtypes = [c_ip, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_ip]
        _gen = L
    return _gen


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def gen_coo(shape, nnz: int, *, zipf_s: float = 0.0, normal_vals: bool = False, seed: int = 12345,
            threads: int = 0):
    """Exact-nnz tensor of the device generator (tk_gen.cu gen_coo), built on the host:
    row-major canonical subs (nnz, d) int64 and float64 vals, byte-identical to
    ``DeviceCoo.generate(shape, nnz, zipf_s=..., normal_vals=..., seed=...)``."""
    shape = tuple(int(s) for s in shape)
    d = len(shape)
    subs = np.empty((nnz, d), dtype=np.int64)
    vals = np.empty(nnz, dtype=np.float64)
    shp = np.asarray(shape, dtype=np.int64)
    rc = gen_lib().tkg_gen_coo(d, _ip(shp), int(nnz), float(zipf_s), int(bool(normal_vals)),
                               int(seed) & (2**64 - 1), int(threads or host_threads()), _ip(subs), _dp(vals))
    if rc != 0:
        raise ValueError(f"gen_coo: bad arguments (rc={rc})")
    return subs, vals


def gen_uniform(n: int, seed: int) -> np.ndarray:
    """The device's seeded uniform vector (tk_gen.cu uniform_kernel), on the host."""
    out = np.empty(int(n), dtype=np.float64)
    gen_lib().tkg_gen_uniform(int(n), int(seed) & (2**64 - 1), _dp(out))
    return out


def shard_bounds(subs, nkeep: int, parts: int) -> list:
    """Split points of row-major canonical ``subs`` into ``parts`` ranges, each moved forward to
    the next change of the first ``nkeep`` columns (no output group spans two ranges)."""
    subs = np.ascontiguousarray(subs, dtype=np.int64)
    b = np.empty(parts + 1, dtype=np.int64)
    gen_lib().tkg_shard_bounds(_ip(subs), subs.shape[0], subs.shape[1], int(nkeep), int(parts), _ip(b))
    return [int(v) for v in b]


def ttv_raw_threads(subs, vals, shape, x, k, threads: int = 0):
    """The reference's compiled ``ttv_raw`` (oracle/_ref; else the C port) over ``threads``
    shards of a canonical tensor cut where the modes before ``k`` change, each shard on
    its own Python thread with the GIL released (``ttv_raw(..., release_gil=True)``,
    _ckernels.pyx:370-374).  The rank-order concatenation is the one-call result.  Returns
    ((subs, vals, shape), seconds, kind)."""
    import time
    from concurrent.futures import ThreadPoolExecutor
    threads = int(threads or host_threads())
    ck = reference_module()
    kind = "reference" if ck is not None else "port"
    # the sorted key prefix of the kept tuple is the modes before k: cut shards where it changes
    if int(k) == 0:
        threads = 1
    bounds = shard_bounds(subs, max(int(k), 1), threads)

    def run(i):
        lo, hi = bounds[i], bounds[i + 1]
        if ck is not None:
            return ck.ttv_raw(subs[lo:hi], vals[lo:hi], tuple(shape), x, k, True)
        return ttv_raw(subs[lo:hi], vals[lo:hi], shape, x, k)
    with ThreadPoolExecutor(threads) as ex:
        t0 = time.perf_counter()
        parts = list(ex.map(run, range(threads)))
        el = time.perf_counter() - t0
    return parts, el, kind


def result_digest(parts) -> dict:
    """sha256 of the concatenated (subs, vals) bytes of a TTV result given as a list of
    (subs, vals, shape) parts in order (one part = a whole result).  Row-major int64 subs and
    float64 vals: the reference's TtvRawResult layout, so GPU and CPU results hash alike."""
    import hashlib
    hs, hv = hashlib.sha256(), hashlib.sha256()
    u = 0
    for s, v, _ in parts:
        hs.update(np.ascontiguousarray(s, dtype=np.int64).data)
        hv.update(np.ascontiguousarray(v, dtype=np.float64).data)
        u += len(v)
    return {"u": u, "subs_sha256": hs.hexdigest(), "vals_sha256": hv.hexdigest()}


def compare_parts(parts, subs, vals) -> bool:
    """Bitwise equality of a result given as ordered parts with one contiguous result."""
    off = 0
    for s, v, _ in parts:
        n = len(v)
        if not np.array_equal(np.asarray(s).reshape(n, -1), subs[off:off + n].reshape(n, -1)):
            return False
        if not np.array_equal(np.asarray(v).view(np.int64), np.asarray(vals[off:off + n]).view(np.int64)):
            return False
        off += n
    return off == len(vals)


def ttv_multi_dense_threads(subs, vals, shape, vecs: dict, keep: int = 0, threads: int = 0):
    """``ttv_multi_dense`` on every host thread: canonical input with ``keep == 0`` is cut into
    key-aligned shards of the keep mode (no keep index spans two shards), each shard runs the
    chain of the reference's ``ttv_raw`` (oracle/_ref, GIL released; else the C port) and
    densifies into its own disjoint part of the output.  Returns (out, seconds, kind)."""
    import time
    from concurrent.futures import ThreadPoolExecutor
    if keep != 0:
        raise ValueError("ttv_multi_dense_threads: keep must be 0 (canonical order sorts mode 0)")
    threads = int(threads or host_threads())
    ck = reference_module()
    kind = "reference" if ck is not None else "port"
    d = len(shape)
    bounds = shard_bounds(subs, 1, threads)
    out = np.zeros(shape[keep], dtype=np.float64)

    def run(i):
        lo, hi = bounds[i], bounds[i + 1]
        if hi <= lo:
            return
        cs, cv, csh = subs[lo:hi], vals[lo:hi], tuple(shape)
        for m in sorted((m for m in range(d) if m != keep), reverse=True):
            if ck is not None:
                cs, cv, csh = ck.ttv_raw(cs, cv, csh, vecs[m], m, True)
            else:
                cs, cv, csh = ttv_raw(cs, cv, csh, vecs[m], m)
        out[np.asarray(cs)[:, 0]] = cv
    with ThreadPoolExecutor(threads) as ex:
        t0 = time.perf_counter()
        list(ex.map(run, range(threads)))
        el = time.perf_counter() - t0
    return out, el, kind
