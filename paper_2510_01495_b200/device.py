"""Device-resident COO tensors (struct-of-arrays in HBM) and the device-level TTV calls.

HBM layout: one int64 column per mode (``cols[m][r] = subs[r, m]``) and one
float64 value column, each its own 16-byte-aligned allocation, rows in canonical
(lexicographic) order.  PyTorch only provides the allocations and the stream; every byte of
arithmetic runs in libtk_b200.so.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import DimensionError


def _stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _to_device(arr: np.ndarray, device) -> torch.Tensor:
    """Device copy of a host array that may be read-only (a SparseCooTensor's arrays are,
    sparse.py:101-107): the host tensor is only ever the source of the copy, so torch's
    non-writable warning does not apply."""
    if not arr.flags.writeable:
        import warnings
        with warnings.catch_warnings():
            warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
            return torch.from_numpy(arr).to(device)
    return torch.from_numpy(arr).to(device)


class DeviceCoo:
    """A d-way COO tensor resident on one GPU, SoA columns + values."""

    def __init__(self, cols, vals, shape):
        self.cols = list(cols)
        self.vals = vals
        self.shape = tuple(int(s) for s in shape)
        if len(self.cols) != len(self.shape):
            raise DimensionError("one column per mode expected")

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def device(self):
        return self.vals.device

    def nbytes(self) -> int:
        return self.nnz * 8 * (self.ndim + 1)

    # ---- construction --------------------------------------------------------------------
    @classmethod
    def from_host(cls, subs, vals, shape, device="cuda"):
        subs = np.asarray(subs, dtype=np.int64).reshape(-1, len(shape))
        cols = [_to_device(np.ascontiguousarray(subs[:, m]), device) for m in range(len(shape))]
        v = _to_device(np.ascontiguousarray(np.asarray(vals, dtype=np.float64)), device)
        return cls(cols, v, shape)

    @classmethod
    def generate(cls, shape, nnz: int, *, zipf_s: float = 0.0, normal_vals: bool = False, seed: int = 12345,
                 device="cuda", stream=None):
        """Exact-nnz synthetic tensor generated on the device (tk_gen_coo_device)."""
        d = len(shape)
        cols = [torch.empty(nnz, dtype=torch.int64, device=device) for _ in range(d)]
        vals = torch.empty(nnz, dtype=torch.float64, device=device)
        _lib.check(_lib.load().tk_gen_coo_device(
            d, _lib.i64_array(shape), nnz, float(zipf_s), int(bool(normal_vals)), int(seed) & (2**64 - 1),
            _lib.ptr_array([c.data_ptr() for c in cols]), vals.data_ptr(), _stream_handle(stream)))
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        return cls(cols, vals, shape)

    def to_host(self):
        subs = torch.stack([c.cpu() for c in self.cols], dim=1).numpy()
        return np.ascontiguousarray(subs), self.vals.cpu().numpy()

    def slice(self, lo: int, hi: int, copy: bool = True) -> "DeviceCoo":
        cols = [c[lo:hi].clone() if copy else c[lo:hi] for c in self.cols]
        vals = self.vals[lo:hi].clone() if copy else self.vals[lo:hi]
        return DeviceCoo(cols, vals, self.shape)

    # ---- kernels -------------------------------------------------------------------------
    def ttv(self, x: torch.Tensor, k: int, out_subs=None, out_vals=None, stream=None):
        """Mode-k TTV on the device.  Returns (u, out_subs[(cap, d-1)], out_vals[cap]); rows
        [0, u) are the canonical result (tk_ttv_f64_device)."""
        d = self.ndim
        if out_subs is None:
            out_subs = torch.empty((max(self.nnz, 1), d - 1), dtype=torch.int64, device=self.device)
        if out_vals is None:
            out_vals = torch.empty(max(self.nnz, 1), dtype=torch.float64, device=self.device)
        u = ctypes.c_int64(0)
        _lib.check(_lib.load().tk_ttv_f64_device(
            d, _lib.i64_array(self.shape), self.nnz, _lib.ptr_array([c.data_ptr() for c in self.cols]), None,
            self.vals.data_ptr(), x.data_ptr(), int(x.shape[0]), int(k), out_subs.data_ptr(),
            out_vals.data_ptr(), ctypes.byref(u), _stream_handle(stream)))
        return u.value, out_subs, out_vals

    def ttv_dense(self, vecs: dict, keep: int, out=None, stream=None):
        """Contract every mode but ``keep``; dense float64[shape[keep]] (tk_ttv_dense_f64_device)."""
        d = self.ndim
        if out is None:
            out = torch.empty(self.shape[keep], dtype=torch.float64, device=self.device)
        ptrs = [0 if m == keep else vecs[m].data_ptr() for m in range(d)]
        _lib.check(_lib.load().tk_ttv_dense_f64_device(
            d, _lib.i64_array(self.shape), self.nnz, _lib.ptr_array([c.data_ptr() for c in self.cols]), None,
            self.vals.data_ptr(), int(keep), _lib.ptr_array(ptrs), out.data_ptr(), _stream_handle(stream)))
        return out


    def ttv_dense_peers(self, vecs: dict, keep: int, outs, key_lo: int, key_hi: int, stream=None):
        """Sharded dense TTV: this shard's result for keep-mode indices [key_lo, key_hi) stored
        into every output copy in ``outs`` (tensors or raw device pointers: this GPU's vector and
        peers' vectors mapped with ``ipc_open``) by the kernel itself (tk_ttv_dense_f64_device_peers)."""
        d = self.ndim
        ptrs = [0 if m == keep else vecs[m].data_ptr() for m in range(d)]
        optrs = [o if isinstance(o, int) else o.data_ptr() for o in outs]
        _lib.check(_lib.load().tk_ttv_dense_f64_device_peers(
            d, _lib.i64_array(self.shape), self.nnz, _lib.ptr_array([c.data_ptr() for c in self.cols]),
            self.vals.data_ptr(), int(keep), _lib.ptr_array(ptrs), _lib.ptr_array(optrs), len(optrs),
            int(key_lo), int(key_hi), _stream_handle(stream)))

    def mttkrp(self, factors: dict, n: int, out=None, stream=None):
        """Mode-``n`` MTTKRP with row-major device factors ``{m: (shape[m], R)}``; dense
        float64[(shape[n], R)] (tk_mttkrp_f64_device)."""
        d = self.ndim
        rank = int(next(iter(factors.values())).shape[1])
        if out is None:
            out = torch.empty((self.shape[n], rank), dtype=torch.float64, device=self.device)
        ptrs = [0 if m == n else factors[m].data_ptr() for m in range(d)]
        _lib.check(_lib.load().tk_mttkrp_f64_device(
            d, _lib.i64_array(self.shape), self.nnz, _lib.ptr_array([c.data_ptr() for c in self.cols]), None,
            self.vals.data_ptr(), int(n), rank, _lib.ptr_array(ptrs), out.data_ptr(), _stream_handle(stream)))
        return out


def uniform_vector(n: int, seed: int, device="cuda", stream=None) -> torch.Tensor:
    out = torch.empty(n, dtype=torch.float64, device=device)
    _lib.check(_lib.load().tk_gen_uniform_device(n, int(seed) & (2**64 - 1), out.data_ptr(), _stream_handle(stream)))
    return out


def dot(x: torch.Tensor, y: torch.Tensor, out: torch.Tensor, stream=None) -> None:
    _lib.check(_lib.load().tk_dot_f64_device(x.data_ptr(), y.data_ptr(), int(x.shape[0]), out.data_ptr(),
                                              _stream_handle(stream)))


def matvec(a: torch.Tensor, x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
    _lib.check(_lib.load().tk_matvec_f64_device(a.data_ptr(), int(a.shape[0]), int(a.shape[1]), x.data_ptr(),
                                                 y.data_ptr(), _stream_handle(stream)))


class IpcVector:
    """A float64 device vector in its own exportable allocation (tk_ipc_alloc), usable as a
    zero-copy torch tensor (``.tensor``) and exportable to peer processes (``.handle()``)."""

    def __init__(self, n: int, device_index: int):
        self.n, self.device_index = int(n), int(device_index)
        p = ctypes.c_void_p()
        _lib.check(_lib.load().tk_ipc_alloc(max(8 * self.n, 8), ctypes.byref(p)))
        self.ptr = int(p.value)
        self.__cuda_array_interface__ = {"shape": (self.n,), "typestr": "<f8", "data": (self.ptr, False),
                                         "version": 3, "strides": None}
        self.tensor = torch.as_tensor(self, device=f"cuda:{self.device_index}")

    def handle(self) -> bytes:
        h = ctypes.create_string_buffer(64)
        _lib.check(_lib.load().tk_ipc_get_handle(self.ptr, h))
        return h.raw

    def free(self) -> None:
        if self.ptr:
            self.tensor = None
            _lib.check(_lib.load().tk_ipc_free(self.ptr))
            self.ptr = 0


def ipc_open(handle: bytes) -> int:
    """Map a peer's exported allocation into this process; returns its device pointer."""
    p = ctypes.c_void_p()
    _lib.check(_lib.load().tk_ipc_open(ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _lib.check(_lib.load().tk_ipc_close(ctypes.c_void_p(ptr)))
