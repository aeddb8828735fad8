"""Sharding of the TTV path across GPUs (one process per GPU, torch.distributed plumbing).

Nonzeros are independent units; the only exchange is the merge of results:

* shards are contiguous ranges of the canonical row order, each split point moved forward
  to the next change of the kept-mode key, so no output group spans two ranks;
* sparse result (configs 3, 5): every rank's output is a canonical slice and the
  rank-order concatenation IS the canonical result, bitwise equal to one GPU; the merge is
  an all-gather of per-rank counts (global offsets), no data moves;
* dense result (config 4): each rank writes only the keep-mode rows it owns into a
  full-length vector (zeros elsewhere) and an all-reduce(sum) merges them -- every element
  has exactly one non-zero contributor, so the sum is exact.

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


def global_offsets(counts) -> list:
    off = [0]
    for c in counts:
        off.append(off[-1] + c)
    return off


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
