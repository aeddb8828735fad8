"""Sharding of the TTV path across GPUs (one process per GPU; the data plane is NCCL inside
libtk_b200.so, torch.distributed only bootstraps the communicator).

Nonzeros are independent units; the only exchange is the merge of results:

* shards are contiguous ranges of the canonical row order, each split point moved forward
  to the next change of the kept-mode key, so no output group spans two ranks;
* sparse result (configs 3, 5): every rank's output is a canonical slice and the
  rank-order concatenation IS the canonical result, bitwise equal to one GPU; the merge is
  an all-gather of per-rank counts (global offsets, ``NcclComm.counts_start``), no data
  moves; ``gather_sparse_to_root`` optionally collects the slices on one rank;
* dense result (config 4): each rank owns the keep-mode indices of its shard.  The B200
  path (``PeerDenseMerge``) has the TTV kernel itself store every owned element -- values,
  and zeros for indices without rows -- into every rank's output vector, mapped over NVLink
  by CUDA IPC (handles exchanged once through the communicator), so one stream-ordered
  barrier completes the merge (no all-reduce of the vector).  ``merge_dense`` keeps the
  all-reduce form (each rank writes only its rows into a zeroed full-length vector; every
  element has exactly one non-zero contributor, so the sum is exact) as the NCCL baseline.

Every function that exchanges data takes a communicator with the ``NcclComm`` interface.  The
host-side logic is exercised on CPU with a gloo-backed stand-in (tests/gloo_comm.py); on a GPU
node ``NcclComm`` runs it over NVLink.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib


def kept_prefix_key(cols, nkeep: int, dims) -> torch.Tensor:
    """Linearised key of the first ``nkeep`` modes (row-major over them), one int64 per row."""
    key = cols[0].clone()
    for m in range(1, nkeep):
        key = key * int(dims[m]) + cols[m]
    return key


def shard_bounds(key: torch.Tensor, world: int) -> list:
    """Split points [0 = b0 <= b1 <= ... <= b_world = n] at key changes.

    ``key`` is non-decreasing (canonical order).  b_i is the first row >= i*n/world whose
    key differs from the key of row (that target - 1), i.e. searchsorted(..., right=True).
    """
    n = int(key.shape[0])
    bounds = [0]
    for i in range(1, world):
        t = (i * n) // world
        if t <= 0:
            b = 0
        elif t >= n:
            b = n
        else:
            prev = key[t - 1:t]
            b = int(torch.searchsorted(key, prev, right=True).item())
        bounds.append(max(b, bounds[-1]))
    bounds.append(n)
    return bounds


def shard_bounds_np(key: np.ndarray, world: int) -> list:
    n = int(key.shape[0])
    bounds = [0]
    for i in range(1, world):
        t = (i * n) // world
        b = 0 if t <= 0 else n if t >= n else int(np.searchsorted(key, key[t - 1], side="right"))
        bounds.append(max(b, bounds[-1]))
    bounds.append(n)
    return bounds


def global_offsets(counts) -> list:
    off = [0]
    for c in counts:
        off.append(off[-1] + c)
    return off


def owned_key_range(key: torch.Tensor, bounds, rank: int, nkeep: int) -> tuple:
    """Keep-mode indices [lo, hi) rank ``rank`` owns for a dense result: from the key of its first
    row (0 for rank 0) to the key of the next rank's first row (``nkeep`` for the last rank).
    ``key`` is the keep-mode column (non-decreasing), ``bounds`` from ``shard_bounds``.  The
    ranges partition [0, nkeep), so every element of the result has exactly one owner."""
    n = int(key.shape[0])
    world = len(bounds) - 1

    def first_key(r):
        if r == 0:
            return 0
        if r >= world or bounds[r] >= n:
            return nkeep
        return int(key[bounds[r]].item())
    lo, hi = first_key(rank), first_key(rank + 1)
    return lo, max(lo, hi)


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _torch_nccl_path():
    """PyTorch's own libnccl (so the process holds one NCCL), if it ships one."""
    try:
        import nvidia.nccl
        for p in nvidia.nccl.__path__:
            f = os.path.join(p, "lib", "libnccl.so.2")
            if os.path.exists(f):
                return f
    except ImportError:
        pass
    return None


class NcclComm:
    """One rank's NCCL communicator inside libtk_b200.so (tk_nccl_*, include/tk_b200.h).

    ``bootstrap`` ships rank 0's 128-byte unique id to every rank; by default it is a
    torch.distributed ``broadcast_object_list`` (the only use of torch.distributed here)."""

    def __init__(self, rank: int, world: int, bootstrap=None):
        self.lib = _lib.load()
        path = _torch_nccl_path()
        _lib.check(self.lib.tk_nccl_load(path.encode() if path else None))
        self.rank, self.world = int(rank), int(world)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(self.lib.tk_nccl_get_unique_id(uid))
        if bootstrap is None:
            bootstrap = _torch_bootstrap
        raw = bootstrap(uid.raw if self.rank == 0 else None)
        uid = ctypes.create_string_buffer(bytes(raw), 128)
        self._comm = ctypes.c_void_p()
        _lib.check(self.lib.tk_nccl_comm_init(uid, self.world, self.rank, ctypes.byref(self._comm)))

    # (a) offsets of the sparse result
    def counts_start(self, count: int, stream=None) -> int:
        t = ctypes.c_int32(0)
        _lib.check(self.lib.tk_nccl_counts_start(self._comm, int(count), _stream(stream), ctypes.byref(t)))
        return t.value

    def counts_wait(self, ticket: int) -> list:
        out = (ctypes.c_int64 * self.world)()
        _lib.check(self.lib.tk_nccl_counts_wait(self._comm, int(ticket), out))
        return [int(v) for v in out]

    def allgather_counts(self, count: int, stream=None) -> list:
        return self.counts_wait(self.counts_start(count, stream))

    # (b) the sparse slices on one rank
    def gather_rows(self, subs: torch.Tensor, vals: torch.Tensor, counts, root: int = 0, stream=None):
        nk = subs.shape[1] if subs.dim() == 2 else 1
        cnt = _lib.i64_array(counts)
        dst_s = dst_v = None
        if self.rank == root:
            total = sum(counts)
            dst_s = torch.empty((max(total, 1), nk), dtype=torch.int64, device=subs.device)
            dst_v = torch.empty(max(total, 1), dtype=torch.float64, device=vals.device)
        _lib.check(self.lib.tk_nccl_gather_rows(
            self._comm, int(root), subs.data_ptr(), vals.data_ptr(), nk, cnt,
            dst_s.data_ptr() if dst_s is not None else None, dst_v.data_ptr() if dst_v is not None else None,
            _stream(stream)))
        if dst_s is None:
            return None, None
        total = sum(counts)
        return dst_s[:total], dst_v[:total]

    # (c) dense merge: IPC handles, barrier, all-reduce baseline
    def allgather_bytes(self, data: bytes) -> list:
        n = len(data)
        dst = ctypes.create_string_buffer(n * self.world)
        _lib.check(self.lib.tk_nccl_allgather_bytes(self._comm, ctypes.create_string_buffer(data, n), dst, n))
        return [dst.raw[r * n:(r + 1) * n] for r in range(self.world)]

    def barrier(self, stream=None) -> None:
        _lib.check(self.lib.tk_nccl_barrier(self._comm, _stream(stream)))

    def allreduce_sum_(self, t: torch.Tensor, stream=None) -> torch.Tensor:
        _lib.check(self.lib.tk_nccl_allreduce_sum_f64(self._comm, t.data_ptr(), int(t.numel()), _stream(stream)))
        return t

    def close(self) -> None:
        if self._comm:
            _lib.check(self.lib.tk_nccl_comm_free(self._comm))
            self._comm = ctypes.c_void_p()


def _torch_bootstrap(uid):
    import torch.distributed as dist
    box = [uid]
    dist.broadcast_object_list(box, src=0)
    return box[0]


def gather_counts(comm, u: int) -> list:
    """All-gather per-rank output counts; returns the list in rank order."""
    return comm.allgather_counts(u)


def gather_sparse_to_root(comm, subs: torch.Tensor, vals: torch.Tensor, counts, root: int = 0):
    """Optional gather of the distributed sparse result to ``root`` (timed separately:
    bounded by the root's link ingress).  Returns (subs, vals) on root."""
    return comm.gather_rows(subs, vals, counts, root)


def merge_dense(comm, out: torch.Tensor) -> torch.Tensor:
    """Sum the per-rank dense partials in place (disjoint supports: exact)."""
    return comm.allreduce_sum_(out)


class PeerDenseMerge:
    """Sharded dense TTV merged by the kernel's own NVLink stores (stage 2).

    Every rank allocates its output vector in an exportable allocation, the 64-byte CUDA IPC
    handles are all-gathered once through the communicator, and each rank maps its peers'
    vectors.  ``run`` launches ``tk_ttv_dense_f64_device_peers`` with all N output pointers and
    the rank's owned key range, then the communicator's stream-ordered barrier (it completes only
    after every rank's kernel, hence every peer store, has finished).  Afterwards every rank's
    ``out`` holds the full result, identical on all ranks.
    """

    def __init__(self, nkeep: int, device_index: int, comm):
        from .device import IpcVector, ipc_open
        self.comm = comm
        self.rank, self.world = comm.rank, comm.world
        self.local = IpcVector(nkeep, device_index)
        handles = comm.allgather_bytes(self.local.handle())
        self.ptrs = [self.local.ptr if r == self.rank else ipc_open(h) for r, h in enumerate(handles)]
        self.device = torch.device(f"cuda:{device_index}")

    @property
    def out(self) -> torch.Tensor:
        return self.local.tensor

    def run(self, dt, vecs: dict, keep: int, key_lo: int, key_hi: int, stream=None) -> torch.Tensor:
        dt.ttv_dense_peers(vecs, keep, self.ptrs, key_lo, key_hi, stream)
        self.comm.barrier(stream)
        return self.out

    def close(self):
        from .device import ipc_close
        torch.cuda.synchronize(self.device)
        self.comm.barrier()  # nobody stores into a mapping that is going away
        torch.cuda.synchronize(self.device)
        for r, p in enumerate(self.ptrs):
            if r != self.rank:
                ipc_close(p)
        self.comm.barrier()
        torch.cuda.synchronize(self.device)
        self.local.free()
