"""N>1 host logic with world_size-2 gloo on CPU: group-aligned shard bounds, count
all-gather / offsets, exact dense merge.  Per-shard results come from the oracle (the
checker) standing in for the per-GPU kernel, so this validates the sharding contract:
rank-order concatenation of shard results == the single-device result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_01495_b200 import multi

from gloo_comm import GlooComm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tensor(seed=3, shape=(40, 30, 50), nnz=6000, zipf=True):
    rng = np.random.default_rng(seed)
    if zipf:
        cols = [np.minimum(rng.zipf(1.3, size=4 * nnz) - 1, n - 1) for n in shape]
        lin = np.ravel_multi_index(cols, shape)
        lin = np.unique(lin)[:nnz]
    else:
        lin = np.unique(rng.integers(0, int(np.prod(shape)), size=nnz))
    subs = np.column_stack(np.unravel_index(lin, shape)).astype(np.int64)
    vals = rng.standard_normal(lin.size)
    return subs, vals, shape


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        subs, vals, shape = _tensor()
        k = 2
        x = np.random.default_rng(9).random(shape[k])
        key = torch.from_numpy(subs[:, 0] * shape[1] + subs[:, 1])
        bounds = multi.shard_bounds(key, world)
        assert bounds == multi.shard_bounds_np(key.numpy(), world)
        lo, hi = bounds[rank], bounds[rank + 1]
        s, v, _ = oracle.ttv_raw(subs[lo:hi], vals[lo:hi], shape, x, k)
        comm = GlooComm()
        counts = multi.gather_counts(comm, len(v))
        off = multi.global_offsets(counts)
        # the pipelined form the bench uses: start step i+1's gather before waiting on step i's
        t1 = comm.counts_start(len(v))
        t2 = comm.counts_start(2 * len(v))
        assert comm.counts_wait(t1) == counts and comm.counts_wait(t2) == [2 * c for c in counts]
        # sparse gather to root (optional path)
        all_s, all_v = multi.gather_sparse_to_root(comm, torch.from_numpy(s.copy()), torch.from_numpy(v.copy()), counts)
        # dense merge: keep mode 0, contract 1 and 2; shards split where the mode-0 index changes
        vecs = {1: np.random.default_rng(5).random(shape[1]), 2: np.random.default_rng(6).random(shape[2])}
        db = multi.shard_bounds(torch.from_numpy(subs[:, 0].copy()), world)
        lo, hi = db[rank], db[rank + 1]
        dense = oracle.ttv_multi_dense(subs[lo:hi], vals[lo:hi], shape, vecs, 0)
        merged = multi.merge_dense(comm, torch.from_numpy(dense.copy())).numpy()
        assert comm.allgather_bytes(bytes([rank]) * 64) == [bytes([r]) * 64 for r in range(world)]
        if rank == 0:
            result_q.put(("ok", bounds, counts, off, all_s.numpy(), all_v.numpy(), merged))
    except Exception as exc:  # pragma: no cover - reported to the parent
        result_q.put(("err", repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_device():
    from oracle import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == "ok", res
    _, bounds, counts, off, all_s, all_v, merged = res
    subs, vals, shape = _tensor()
    k = 2
    x = np.random.default_rng(9).random(shape[k])
    s, v, _ = oracle.ttv_raw(subs, vals, shape, x, k)
    # boundaries fall on key changes, so no group is split
    key = subs[:, 0] * shape[1] + subs[:, 1]
    b = bounds[1]
    assert 0 < b < len(key) and key[b] != key[b - 1]
    assert off[-1] == len(v) == sum(counts)
    assert all_s.tobytes() == s.tobytes() and all_v.tobytes() == v.tobytes()
    vecs = {1: np.random.default_rng(5).random(shape[1]), 2: np.random.default_rng(6).random(shape[2])}
    full = oracle.ttv_multi_dense(subs, vals, shape, vecs, 0)
    assert merged.tobytes() == full.tobytes()


def test_shard_bounds_edge_cases():
    key = torch.tensor([0, 0, 0, 0, 1, 1, 2, 2, 2, 2])
    assert multi.shard_bounds(key, 1) == [0, 10]
    b = multi.shard_bounds(key, 4)
    assert b[0] == 0 and b[-1] == 10 and b == sorted(b)
    for x in b[1:-1]:
        assert x in (0, 4, 6, 10)
    # a single huge group cannot be split: everything lands on one rank
    assert multi.shard_bounds(torch.zeros(8, dtype=torch.int64), 3) == [0, 8, 8, 8]
    assert multi.shard_bounds(torch.zeros(0, dtype=torch.int64), 2) == [0, 0, 0]


def test_owned_key_ranges_partition_the_keep_mode():
    """Dense-result ownership (PeerDenseMerge): the ranks' [lo, hi) ranges tile [0, nkeep) and
    every key of a shard lies in its own rank's range, including empty shards and keys without
    rows at either end."""
    rng = np.random.default_rng(4)
    for trial in range(40):
        nkeep = int(rng.integers(1, 30))
        n = int(rng.integers(0, 200))
        key = torch.from_numpy(np.sort(rng.integers(0, nkeep, size=n)))
        for world in (1, 2, 3, 5, 8):
            bounds = multi.shard_bounds(key, world)
            ranges = [multi.owned_key_range(key, bounds, r, nkeep) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == nkeep
            for r in range(world - 1):
                assert ranges[r][1] == ranges[r + 1][0]
            for r in range(world):
                lo, hi = ranges[r]
                ks = key[bounds[r]:bounds[r + 1]]
                assert lo <= hi
                if ks.numel():
                    assert lo <= int(ks.min()) and int(ks.max()) < hi
