"""Sharding of the TTV path across GPUs (one process per GPU, torch.distributed plumbing).

Nonzeros are independent units; the only exchange is the merge of results:

* shards are contiguous ranges of the canonical row order, each split point moved forward
  to the next change of the kept-mode key, so no output group spans two ranks;
* sparse result (configs 3, 5): every rank's output is a canonical slice and the
  rank-order concatenation IS the canonical result, bitwise equal to one GPU; the merge is
  an all-gather of per-rank counts (global offsets), no data moves;
* dense result (config 4): each rank owns the keep-mode indices of its shard.  The B200
  path (``PeerDenseMerge``) has the TTV kernel itself store every owned element -- values,
  and zeros for indices without rows -- into every rank's output vector, mapped over NVLink
  by CUDA IPC, so one stream-ordered barrier completes the merge (no all-reduce of the
  vector).  ``merge_dense`` keeps the all-reduce form (each rank writes only its rows into a
  zeroed full-length vector; every element has exactly one non-zero contributor, so the sum
  is exact) as the NCCL baseline.

The host-side logic here is exercised with gloo on CPU (tests/test_multi_cpu.py); on the
GPU box the same calls run over NCCL.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


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


def gather_counts(u: int, device) -> list:
    """All-gather per-rank output counts; returns the list in rank order."""
    world = dist.get_world_size()
    t = torch.tensor([u], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [int(v.item()) for v in out]


def gather_counts_async(u: int, device):
    """Start the all-gather of per-rank output counts without waiting for it (the next step's
    TTV kernel runs while it completes); finish with ``wait_counts``."""
    world = dist.get_world_size()
    t = torch.tensor([u], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    return dist.all_gather(out, t, async_op=True), out


def wait_counts(handle) -> list:
    work, out = handle
    work.wait()
    return [int(v.item()) for v in out]


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


class PeerDenseMerge:
    """Sharded dense TTV merged by the kernel's own NVLink stores (stage 2).

    Every rank allocates its output vector in an exportable allocation, the 64-byte CUDA IPC
    handles are all-gathered once, and each rank maps its peers' vectors.  ``run`` launches
    ``tk_ttv_dense_f64_device_peers`` with all N output pointers and the rank's owned key range,
    then a stream-ordered barrier (a one-element all-reduce: it completes only after every
    rank's kernel, hence every peer store, has finished).  Afterwards every rank's ``out`` holds
    the full result, identical on all ranks.
    """

    def __init__(self, nkeep: int, device_index: int):
        from .device import IpcVector, ipc_open
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.local = IpcVector(nkeep, device_index)
        handles = [None] * self.world
        dist.all_gather_object(handles, self.local.handle())
        self.ptrs = [self.local.ptr if r == self.rank else ipc_open(h) for r, h in enumerate(handles)]
        self.device = torch.device(f"cuda:{device_index}")
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)

    @property
    def out(self) -> torch.Tensor:
        return self.local.tensor

    def run(self, dt, vecs: dict, keep: int, key_lo: int, key_hi: int, stream=None) -> torch.Tensor:
        dt.ttv_dense_peers(vecs, keep, self.ptrs, key_lo, key_hi, stream)
        self.barrier()
        return self.out

    def barrier(self):
        if dist.get_backend() == "nccl":
            dist.all_reduce(self._flag)  # stream-ordered behind the kernel on every rank
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier()

    def close(self):
        from .device import ipc_close
        torch.cuda.synchronize(self.device)
        dist.barrier()  # nobody stores into a mapping that is going away
        for r, p in enumerate(self.ptrs):
            if r != self.rank:
                ipc_close(p)
        dist.barrier()
        self.local.free()


def merge_dense(out: torch.Tensor) -> torch.Tensor:
    """Sum the per-rank dense partials in place (disjoint supports: exact)."""
    dist.all_reduce(out, op=dist.ReduceOp.SUM)
    return out


def gather_sparse_to_root(subs: torch.Tensor, vals: torch.Tensor, counts, root: int = 0):
    """Optional gather of the distributed sparse result to ``root`` (timed separately:
    bounded by the root's link ingress).  Returns (subs, vals) on root."""
    rank, world = dist.get_rank(), dist.get_world_size()
    nk = subs.shape[1] if subs.dim() == 2 else 1
    if rank == root:
        total = sum(counts)
        all_s = torch.empty((total, nk), dtype=subs.dtype, device=subs.device)
        all_v = torch.empty(total, dtype=vals.dtype, device=vals.device)
        off = global_offsets(counts)
        for r in range(world):
            if r == root:
                all_s[off[r]:off[r + 1]].copy_(subs[:counts[r]])
                all_v[off[r]:off[r + 1]].copy_(vals[:counts[r]])
            elif counts[r]:
                dist.recv(all_s[off[r]:off[r + 1]], src=r)
                dist.recv(all_v[off[r]:off[r + 1]], src=r)
        return all_s, all_v
    if counts[rank]:
        dist.send(subs[:counts[rank]].contiguous(), dst=root)
        dist.send(vals[:counts[rank]].contiguous(), dst=root)
    return None, None
