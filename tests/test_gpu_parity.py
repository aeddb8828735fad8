"""GPU parity: the sm_100a path through the C ABI against the CPU oracle and the
reference's golden vectors.  Bar: coordinates bit-exact; TTV values bit-exact (serial
in-group folds, the reference's exact operation order); dot / matvec / dense
multi-vector TTV within 1e-12 relative (north-star tolerance, written per test)."""

import hashlib
import os
import sys

import numpy as np
import pytest

from conftest import ttv_cases

pytestmark = pytest.mark.gpu

REL = 1e-12  # north-star FP64 tolerance for tree-order reductions


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def K():
    from paper_2510_01495_b200 import _lib, backend
    assert _lib.device_count() > 0, "no CUDA device visible"
    return backend.kernels()


def assert_ttv_equal(got, exp, name=""):
    s, v, sh = got
    assert tuple(sh) == tuple(exp[2]), name
    assert np.asarray(s).shape == np.asarray(exp[0]).shape, name
    assert np.asarray(s).tobytes() == np.asarray(exp[0]).tobytes(), name
    assert np.asarray(v).tobytes() == np.asarray(exp[1]).tobytes(), name


def test_golden_ttv_cases_bit_exact(K, golden_small, golden_hashes):
    from paper_2510_01495_b200 import errors
    for name, subs, vals, shape, x, k, err, exp in ttv_cases(golden_small, golden_hashes):
        if err:
            with pytest.raises(getattr(errors, err)):
                K.ttv_raw(subs, vals, shape, x, k)
            continue
        assert_ttv_equal(K.ttv_raw(subs, vals, shape, x, k), exp, name)


def test_golden_dense_cases(K, golden_small, golden_hashes):
    for i in range(golden_hashes["dense_cases"]):
        a, x, y = golden_small[f"d{i}_a"], golden_small[f"d{i}_x"], golden_small[f"d{i}_y"]
        np.testing.assert_allclose(K.matvec(a, x), golden_small[f"d{i}_mv"], rtol=REL, atol=0)
        np.testing.assert_allclose(K.dot(x, y), golden_small[f"d{i}_dot"], rtol=REL, atol=0)


def test_dense_pinned_examples_exact():
    import paper_2510_01495_b200 as tk
    assert tk.dot([1.0, 2.0, 3.0], [4.0, 5.0, 6.0]) == 32.0
    assert tk.dot([], []) == 0.0
    assert tk.dot([0.0, 0.0, 0.0], [5.0, 5.0, 5.0]) == 0.0
    y = np.random.default_rng(3).random(6)
    for i in range(6):
        e = np.zeros(6)
        e[i] = 1.0
        assert np.float64(tk.dot(e, y)).tobytes() == np.float64(y[i]).tobytes()
    assert np.array_equal(tk.matvec(np.eye(2), [3.0, 7.0]), [3.0, 7.0])
    assert np.array_equal(tk.matvec([[1.0, 2.0], [3.0, 4.0]], [1.0, 1.0]), [3.0, 7.0])
    assert tk.matvec(np.zeros((0, 3)), [1.0, 1.0, 1.0]).shape == (0,)
    assert np.array_equal(tk.matvec(np.zeros((2, 0)), []), [0.0, 0.0])
    assert tk.dot([1, 2], [3, 4]) == 11.0


def test_config1_dot_full_size(K, oracle, golden_hashes):
    from paper_2510_01495_b200 import synth
    ops = synth.host_operands(1)
    ref = float.fromhex(golden_hashes["cfg1"]["dot_hex"])
    got = K.dot(ops["x"], ops["y"])
    assert abs(got - ref) <= REL * abs(ref)
    for n in (1, 2, 3, 17, 1023, 4097, 100001, 2_400_001, 10_000_000):
        x, y = np.random.default_rng(n).random(n), np.random.default_rng(n + 1).random(n)
        r = oracle.dot(x, y)
        assert abs(K.dot(x, y) - r) <= REL * abs(r)
    # unaligned views take the scalar path
    x = np.random.default_rng(5).random(1001)
    assert abs(K.dot(x[1:], x[:-1]) - oracle.dot(x[1:], x[:-1])) <= REL * oracle.dot(x[1:], x[:-1])


def test_config2_matvec_full_size(K, oracle):
    from paper_2510_01495_b200 import synth
    ops = synth.host_operands(2)
    ref = oracle.matvec(ops["a"], ops["x"])
    np.testing.assert_allclose(K.matvec(ops["a"], ops["x"]), ref, rtol=REL, atol=0)
    for rows, cols in ((1, 1), (7, 3), (33, 65), (100, 4097), (3000, 1)):
        rng = np.random.default_rng(rows * 7 + cols)
        a, x = rng.random((rows, cols)), rng.random(cols)
        np.testing.assert_allclose(K.matvec(a, x), oracle.matvec(a, x), rtol=REL, atol=0)


def test_config3_full_size_matches_reference_hashes(K, golden_hashes):
    from paper_2510_01495_b200 import synth
    ops = synth.host_operands(3)
    t, g = ops["tensor"], golden_hashes["cfg3"]
    s, v, sh = K.ttv_raw(t.subs, t.vals, t.shape, ops["x"], ops["k0"])
    assert len(v) == g["u"] and sha(s) == g["out_subs"] and sha(v) == g["out_vals"]
    assert list(sh) == g["out_shape"]
    g1 = golden_hashes["cfg3_k1"]  # the paper's own middle-mode protocol: the sort path
    s, v, _ = K.ttv_raw(t.subs, t.vals, t.shape, ops["x"], 1)
    assert len(v) == g1["u"] and sha(s) == g1["out_subs"] and sha(v) == g1["out_vals"]


def _random_tensor(rng, shape, nnz, normal=True, zipf=None):
    if zipf:
        cols = [np.minimum(rng.zipf(zipf, size=3 * nnz) - 1, n - 1) for n in shape]
        lin = np.unique(np.ravel_multi_index(cols, shape))[:nnz]
    else:
        lin = np.unique(rng.integers(0, int(np.prod(shape)), size=nnz))
    subs = np.column_stack(np.unravel_index(lin, shape)).astype(np.int64)
    vals = rng.standard_normal(lin.size) if normal else rng.random(lin.size)
    return subs, vals


@pytest.mark.parametrize("shape,nnz,zipf", [
    ((50, 40, 30), 20000, None),
    ((2000, 300, 700), 300000, None),
    ((3000, 2000, 5000), 400000, 1.2),      # skewed: long groups, spills across tiles
    ((7, 9), 50, None),                      # order 2
    ((6, 5, 4, 3, 7), 2000, None),           # order 5
    ((3, 3, 3, 3, 3, 3, 3, 3, 3), 4000, None),  # order 9: runtime-width key kernels
])
def test_random_all_modes_bit_exact(K, oracle, shape, nnz, zipf):
    rng = np.random.default_rng(sum(shape) + nnz)
    subs, vals = _random_tensor(rng, shape, nnz, zipf=zipf)
    for k in range(len(shape)):
        x = rng.standard_normal(shape[k])
        assert_ttv_equal(K.ttv_raw(subs, vals, shape, x, k), oracle.ttv_raw(subs, vals, shape, x, k),
                         f"{shape} k={k}")


def test_single_group_spanning_many_tiles(K, oracle):
    # one kept key, 300k rows: the CTA-cooperative spill fold over ~150 tiles
    n = 300000
    subs = np.column_stack([np.zeros(n), np.zeros(n), np.arange(n)]).astype(np.int64)
    vals = np.random.default_rng(11).standard_normal(n)
    x = np.random.default_rng(12).standard_normal(n)
    assert_ttv_equal(K.ttv_raw(subs, vals, (1, 1, n), x, 2), oracle.ttv_raw(subs, vals, (1, 1, n), x, 2))
    # groups of length 2047..2049 straddling tile edges
    lens = np.tile([2047, 2048, 2049, 1, 4096], 20)
    i0 = np.repeat(np.arange(lens.size), lens)
    i2 = np.concatenate([np.arange(L) for L in lens])
    subs = np.column_stack([i0, np.zeros_like(i0), i2]).astype(np.int64)
    vals = np.random.default_rng(13).standard_normal(i0.size)
    shape = (lens.size, 1, 4096)
    x = np.random.default_rng(14).standard_normal(4096)
    assert_ttv_equal(K.ttv_raw(subs, vals, shape, x, 2), oracle.ttv_raw(subs, vals, shape, x, 2))


@pytest.mark.parametrize("tail", ["stream_goes_on", "stream_ends"])
def test_spill_ring_chunk_boundaries(K, oracle, tail):
    """The open group's spill ring (128-row chunks past the 768+32-row stage, 6 slots, warps 1-3
    producing, warp 0 folding): the group headed at row 700 of tile 0 ends exactly at, one
    before and one after every chunk boundary up to 9 chunks past the stage (wrapping the ring
    once), with the stream going on afterwards or ending with the group."""
    stage = 768 + 32
    for k in range(0, 10):
        for delta in (-1, 0, 1):
            end = stage + 128 * k + delta  # first row after the open group
            if end <= 700:
                continue
            lens = [700, end - 700]
            if tail == "stream_goes_on":
                lens += [1, 3, 130, 2, 900]
            lens = np.array(lens)
            i0 = np.repeat(np.arange(lens.size), lens)
            i2 = np.concatenate([np.arange(L) for L in lens])
            subs = np.column_stack([i0, np.zeros_like(i0), i2]).astype(np.int64)
            vals = np.random.default_rng(k * 7 + delta + 2).standard_normal(i0.size)
            shape = (lens.size, 1, int(lens.max()))
            x = np.random.default_rng(k + 40).standard_normal(shape[2])
            assert_ttv_equal(K.ttv_raw(subs, vals, shape, x, 2), oracle.ttv_raw(subs, vals, shape, x, 2),
                             f"k={k} delta={delta} {tail}")


def test_exact_zero_groups_compacted(K, oracle):
    # +v / -v pairs in the same group cancel exactly; scattered through many tiles
    rng = np.random.default_rng(21)
    g = 100000
    base = rng.standard_normal(g)
    cancel = rng.random(g) < 0.3
    i0 = np.repeat(np.arange(g), 2)
    i2 = np.tile([0, 1], g)
    vals = np.empty(2 * g)
    vals[0::2] = base
    vals[1::2] = np.where(cancel, -base, rng.standard_normal(g))
    subs = np.column_stack([i0, np.zeros_like(i0), i2]).astype(np.int64)
    x = np.ones(2)
    got = K.ttv_raw(subs, vals, (g, 1, 2), x, 2)
    exp = oracle.ttv_raw(subs, vals, (g, 1, 2), x, 2)
    assert len(exp[1]) == g - cancel.sum()
    assert_ttv_equal(got, exp)


def test_unsorted_and_duplicate_raw_buffers(K, oracle):
    rng = np.random.default_rng(31)
    subs = rng.integers(0, 40, size=(50000, 3)).astype(np.int64)
    vals = rng.standard_normal(50000)
    for k in range(3):
        x = rng.standard_normal(40)
        assert_ttv_equal(K.ttv_raw(subs, vals, (40, 40, 40), x, k), oracle.ttv_raw(subs, vals, (40, 40, 40), x, k))


def test_garbage_kept_indices_do_not_crash_and_match(K, oracle):
    from paper_2510_01495_b200 import errors
    rng = np.random.default_rng(41)
    subs = rng.integers(-10**12, 10**12, size=(5000, 3)).astype(np.int64)
    subs[:, 2] = rng.integers(0, 4, size=5000)
    vals = rng.standard_normal(5000)
    x = rng.standard_normal(4)
    assert_ttv_equal(K.ttv_raw(subs, vals, (4, 4, 4), x, 2), oracle.ttv_raw(subs, vals, (4, 4, 4), x, 2))
    subs[17, 2] = 4  # contracted-mode index outside x: must raise, never read out of bounds
    with pytest.raises(errors.DimensionError, match="index out of range"):
        K.ttv_raw(subs, vals, (4, 4, 4), x, 2)


def test_public_api_and_canonicalisation_on_device():
    import paper_2510_01495_b200 as tk
    t = tk.SparseCooTensor([[1, 1], [0, 0], [1, 1], [0, 1]], [2.0, 1.0, 3.0, 0.0], (2, 2))
    assert t.subs.tolist() == [[0, 0], [1, 1]] and t.vals.tolist() == [1.0, 5.0]
    assert tk.SparseCooTensor([[0, 0], [0, 0]], [1.5, -1.5], (2, 2)).nnz == 0
    res = tk.ttv(tk.SparseCooTensor([[0, 0, 0], [0, 1, 0]], [2.0, 3.0], (2, 2, 2)), [10.0, 100.0], 1)
    assert isinstance(res, tk.TtvRawResult)
    assert res.to_tensor() == tk.SparseCooTensor([[0, 0]], [320.0], (2, 2))
    u, s = tk.unique_rows_accumulate([[0, 0], [0, 0], [1, 2]], [1.0, 2.0, 3.0])
    assert u.tolist() == [[0, 0], [1, 2]] and s.tolist() == [3.0, 3.0]
    _, s = tk.unique_rows_accumulate([[0], [0], [0]], [1e16, 1.0, -1e16])
    assert s[0] == ((1e16 + 1.0) + -1e16)
    u, s = tk.unique_rows_accumulate([], [])
    assert u.shape[0] == 0 and s.shape == (0,)
    keys = np.array([[3, 1], [0, 2], [2, 0]])
    w = np.array([0.1, 0.2, 0.3])
    u, s = tk.unique_rows_accumulate(keys, w)
    assert u.tolist() == [[0, 2], [2, 0], [3, 1]] and s.tolist() == [0.2, 0.3, 0.1]


def test_unique_rows_accumulate_matches_reference_pykernels_semantics(oracle):
    import paper_2510_01495_b200 as tk
    rng = np.random.default_rng(51)
    for _ in range(10):
        n = int(rng.integers(1, 3000))
        keys = rng.integers(-3, 4, size=(n, 3))
        w = rng.standard_normal(n)
        u, s = tk.unique_rows_accumulate(keys, w)
        # oracle: TTV with an appended singleton contracted mode keeps the order, but drops
        # zero sums; compare on the nonzero groups and the full key set
        order = np.lexsort(keys.T[::-1])
        ks = keys[order]
        first = np.ones(n, dtype=bool)
        first[1:] = (ks[1:] != ks[:-1]).any(axis=1)
        assert np.array_equal(u, ks[first])
        exp = []
        for i in np.flatnonzero(first):  # the reference: acc = 0.0, then every weight in row order
            j = i
            acc = 0.0
            while j < n and (j == i or not first[j]):
                acc += w[order[j]]
                j += 1
            exp.append(acc)
        assert np.asarray(exp).tobytes() == s.tobytes()
    # all-(-0.0) groups: the reference's fold from +0.0 gives +0.0
    u, s = tk.unique_rows_accumulate([[1], [1], [2], [3], [3]], [-0.0, -0.0, -0.0, 5.0, -5.0])
    assert u.tolist() == [[1], [2], [3]]
    assert np.asarray([0.0, 0.0, 0.0]).tobytes() == s.tobytes()
    if os.path.isdir(os.path.join(oracle.REF_DIR, "tenkern")):
        sys.path.insert(0, oracle.REF_DIR)
        from tenkern import _pykernels
        for keys, w in (([[1], [1], [2]], [-0.0, -0.0, 0.5]), (rng.integers(0, 3, size=(200, 2)), rng.standard_normal(200))):
            ru, rs = _pykernels.unique_rows_accumulate(np.asarray(keys, dtype=np.int64), np.asarray(w, dtype=np.float64))
            gu, gs = tk.unique_rows_accumulate(keys, w)
            assert np.asarray(ru).tolist() == gu.tolist()
            assert np.asarray(rs, dtype=np.float64).tobytes() == gs.tobytes()


def test_timed_entry_points(K):
    x, y = np.random.default_rng(1).random(1000), np.random.default_rng(2).random(1000)
    v, el = K.dot_timed(x, y)
    assert v == K.dot(x, y) and el > 0
    a = np.random.default_rng(3).random((40, 25))
    out, el = K.matvec_timed(a, y[:25])
    assert out.tobytes() == K.matvec(a, y[:25]).tobytes() and el > 0
    import paper_2510_01495_b200 as tk
    t = tk.gen_sparse3(tk.GenSpec(4, "sparse3", (15, 15, 15), 0.1))
    (s, v, sh), el = K.ttv_timed(t.subs, t.vals, t.shape, x[:15], 1)
    s2, v2, sh2 = K.ttv_raw(t.subs, t.vals, t.shape, x[:15], 1)
    assert s.tobytes() == s2.tobytes() and v.tobytes() == v2.tobytes() and sh == sh2 and el > 0
    # release_gil positional flag accepted (BoundKernelSet passes it positionally)
    assert K.dot(x, y, True) == K.dot(x, y)


def test_device_generator_and_device_ttv(oracle):
    import torch
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    shape = (20000, 5000, 1000)
    t = DeviceCoo.generate(shape, 2_000_000, zipf_s=1.2, normal_vals=True, seed=99)
    subs, vals = t.to_host()
    assert subs.shape == (2_000_000, 3) and (vals != 0).all()
    lin = np.ravel_multi_index(subs.T, shape)
    assert (np.diff(lin) > 0).all()  # canonical: sorted, unique
    t2 = DeviceCoo.generate(shape, 2_000_000, zipf_s=1.2, normal_vals=True, seed=99)
    assert torch.equal(t2.cols[0], t.cols[0]) and torch.equal(t2.vals, t.vals)  # deterministic
    x = uniform_vector(shape[2], 7)
    u, os_, ov = t.ttv(x, 2)
    s, v, _ = oracle.ttv_raw(subs, vals, shape, x.cpu().numpy(), 2)
    assert u == len(v)
    assert os_[:u].cpu().numpy().tobytes() == s.tobytes()
    assert ov[:u].cpu().numpy().tobytes() == v.tobytes()


def test_dense_multi_vector_ttv(oracle):
    import torch
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    shape = (2000, 2000, 2000, 2000)
    t = DeviceCoo.generate(shape, 1_000_000, seed=5)
    vecs = {m: uniform_vector(shape[m], 100 + m) for m in (1, 2, 3)}
    out = t.ttv_dense(vecs, 0).cpu().numpy()
    subs, vals = t.to_host()
    ref = oracle.ttv_multi_dense(subs, vals, shape, {m: v.cpu().numpy() for m, v in vecs.items()}, 0)
    nz = ref != 0
    assert np.array_equal(out != 0, nz)
    assert np.max(np.abs(out[nz] - ref[nz]) / np.abs(ref[nz])) <= REL
    # keep != 0: the chained device path, bit-exact with the chained oracle
    vecs0 = {m: uniform_vector(shape[m], 200 + m) for m in (0, 2, 3)}
    out1 = t.ttv_dense(vecs0, 1).cpu().numpy()
    ref1 = oracle.ttv_multi_dense(subs, vals, shape, {m: v.cpu().numpy() for m, v in vecs0.items()}, 1)
    assert out1.tobytes() == ref1.tobytes()
    # a small-valued case across many tiles with long runs
    small = DeviceCoo.generate((4, 50, 60, 70), 200000, seed=6)
    vv = {m: uniform_vector(small.shape[m], 300 + m) for m in (1, 2, 3)}
    o = small.ttv_dense(vv, 0).cpu().numpy()
    s2, v2 = small.to_host()
    r = oracle.ttv_multi_dense(s2, v2, small.shape, {m: v.cpu().numpy() for m, v in vv.items()}, 0)
    assert np.max(np.abs(o - r) / np.abs(r)) <= REL


def _host_ttv(subs, vals, shape, x, k):
    """tk_ttv_f64_host straight through the C ABI (the pipelined path for k == d-1, >= 32M rows)."""
    import ctypes
    from paper_2510_01495_b200 import _lib
    n, d = subs.shape
    os_ = np.empty((n, d - 1), dtype=np.int64)
    ov = np.empty(n, dtype=np.float64)
    u = ctypes.c_int64(0)
    _lib.check(_lib.load().tk_ttv_f64_host(d, _lib.i64_array(shape), n, subs.ctypes.data, vals.ctypes.data,
                                           x.ctypes.data, len(x), k, os_.ctypes.data, ov.ctypes.data,
                                           ctypes.byref(u)))
    return os_[:u.value], ov[:u.value]


def test_host_pipeline_chunks_match_device_path():
    """>= 32M rows, k == d-1: the host call runs in key-aligned chunks with overlapped copies;
    the result must be bit-identical to the one-shot device path (itself oracle-checked)."""
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    shape = (200000, 3000, 5000)
    t = DeviceCoo.generate(shape, 40_000_000, zipf_s=1.2, normal_vals=True, seed=2024)
    x = uniform_vector(shape[2], 11)
    u, os_d, ov_d = t.ttv(x, 2)
    subs, vals = t.to_host()
    s, v = _host_ttv(np.ascontiguousarray(subs), np.ascontiguousarray(vals), shape, x.cpu().numpy(), 2)
    assert len(v) == u
    assert s.tobytes() == os_d[:u].cpu().numpy().tobytes()
    assert v.tobytes() == ov_d[:u].cpu().numpy().tobytes()


def test_host_pipeline_declines_unsorted_and_reports_index_errors():
    from paper_2510_01495_b200 import errors
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    shape = (100000, 3000, 5000)
    t = DeviceCoo.generate(shape, 34_000_000, zipf_s=1.1, normal_vals=True, seed=77)
    x = uniform_vector(shape[2], 3)
    u, os_d, ov_d = t.ttv(x, 2)
    subs, vals = t.to_host()
    subs = np.ascontiguousarray(subs)
    vals = np.ascontiguousarray(vals)
    # reversed row order: not in kept-key order -> the pipelined path declines, the sort path runs
    rs, rv = subs[::-1].copy(), vals[::-1].copy()
    s, v = _host_ttv(rs, rv, shape, x.cpu().numpy(), 2)
    assert len(v) == u and s.tobytes() == os_d[:u].cpu().numpy().tobytes()
    # the reference folds in original row order: reversed input folds each group in reverse
    # order, so compare against the device path on the same reversed rows
    tr = DeviceCoo.from_host(rs, rv, shape)
    u2, _, ov2 = tr.ttv(x, 2)
    assert v.tobytes() == ov2[:u2].cpu().numpy().tobytes()
    # an out-of-range contracted index in a late chunk -> DimensionError, like the reference
    bad = subs.copy()
    bad[-5, 2] = shape[2]
    with pytest.raises(errors.DimensionError):
        _host_ttv(bad, vals, shape, x.cpu().numpy(), 2)


def test_host_pipeline_pinned_and_unpackable_chunks(oracle):
    """The pipelined host call with (a) pinned caller buffers (direct DMA, no staging) and
    (b) pageable buffers whose first chunk holds a negative kept index (no packed form: that chunk
    travels as raw int64 rows) -- both bit-exact against the oracle."""
    import torch
    shape = (300000, 2000, 3000)
    subs, vals = oracle.gen_coo(shape, 20_000_000, zipf_s=1.1, normal_vals=True, seed=31)
    x = oracle.gen_uniform(shape[2], 8)
    es, ev, _ = oracle.ttv_raw(subs, vals, shape, x, 2)
    ps = torch.from_numpy(subs).pin_memory()
    pv = torch.from_numpy(vals).pin_memory()
    s, v = _host_ttv(ps.numpy(), pv.numpy(), shape, x, 2)
    assert s.tobytes() == es.tobytes() and v.tobytes() == ev.tobytes()
    g = subs.copy()
    g[0, 0] = -7  # still lexicographically first: garbage kept index, canonical order kept
    es2, ev2, _ = oracle.ttv_raw(g, vals, shape, x, 2)
    s2, v2 = _host_ttv(g, vals, shape, x, 2)
    assert s2.tobytes() == es2.tobytes() and v2.tobytes() == ev2.tobytes()


def test_pooled_pinned_results_do_not_alias(oracle, tmp_path):
    """Results >= 64 MB come from the library's cached pinned blocks (the D2H writes the caller's
    arrays directly).  A block stays live while any view of it does: a second call made while the
    first result is held must get different memory; a dropped result's block is reused.  With the
    cache disabled (TK_HOST_POOL_MB=0) the results are ordinary owned arrays, bit-identical."""
    import subprocess
    import paper_2510_01495_b200 as tk
    K = tk.kernels()
    shape = (300000, 2000, 3000)
    subs, vals = oracle.gen_coo(shape, 20_000_000, zipf_s=1.1, normal_vals=True, seed=41)
    x2 = oracle.gen_uniform(shape[2], 5)
    x0 = oracle.gen_uniform(shape[0], 6)
    es, ev, _ = oracle.ttv_raw(subs, vals, shape, x2, 2)
    r1 = K.ttv_raw(subs, vals, shape, x2, 2)  # pipelined host path
    assert not r1[1].flags.owndata and r1[1].flags.writeable and r1[0].flags.c_contiguous
    assert r1[0].tobytes() == es.tobytes() and r1[1].tobytes() == ev.tobytes()
    r2 = K.ttv_raw(subs, vals, shape, x2, 2)
    assert not np.shares_memory(r1[1], r2[1]) and not np.shares_memory(r1[0], r2[0])
    assert r1[1].tobytes() == ev.tobytes() and r2[1].tobytes() == ev.tobytes()
    r2[1][:] = 0.0  # the caller owns its result
    assert r1[1].tobytes() == ev.tobytes()
    del r1, r2
    fs, fv, _ = oracle.ttv_raw(subs, vals, shape, x0, 0)
    r3 = K.ttv_raw(subs, vals, shape, x0, 0)  # one-shot host path, direct D2H into the block
    assert r3[0].tobytes() == fs.tobytes() and r3[1].tobytes() == fv.tobytes()
    np.save(tmp_path / "s.npy", subs)
    np.save(tmp_path / "v.npy", vals)
    np.save(tmp_path / "x.npy", x2)
    code = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[2]); import paper_2510_01495_b200 as tk; "
        "p = sys.argv[1]; s = np.load(p + '/s.npy'); v = np.load(p + '/v.npy'); x = np.load(p + '/x.npy'); "
        f"r = tk.kernels().ttv_raw(s, v, {shape!r}, x, 2); assert r[0].flags.owndata and r[1].flags.owndata; "
        "np.save(p + '/rs.npy', r[0]); np.save(p + '/rv.npy', r[1])")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TK_HOST_POOL_MB="0")
    subprocess.run([sys.executable, "-c", code, str(tmp_path), repo], env=env, check=True, timeout=600)
    assert np.load(tmp_path / "rs.npy").tobytes() == es.tobytes()
    assert np.load(tmp_path / "rv.npy").tobytes() == ev.tobytes()


def _canonical_coo(shape, nnz, seed):
    """Distinct uniform coordinates in canonical (lexicographic) order, positive values."""
    rng = np.random.default_rng(seed)
    total = int(np.prod(np.asarray(shape, dtype=np.float64)))
    lin = np.unique(rng.integers(0, total, size=nnz, dtype=np.int64))
    subs = np.stack(np.unravel_index(lin, shape), axis=1).astype(np.int64)
    vals = rng.random(len(lin)) + 0.5
    return np.ascontiguousarray(subs), vals


@pytest.mark.parametrize("shape,nnz", [
    ((5000, 3, 3, 3), 20000),        # runs of ~4 rows: several heads in most 64-row sub-blocks
    ((300, 40, 50), 700000),         # runs of ~2300 rows: cross the 2048-row span boundaries
    ((1, 700, 800), 150000),         # one run over ~73 spans
    ((64, 100), 3000),               # order 2 (a dense matvec-like contraction)
    ((40, 6, 7, 8, 9), 50000),       # order 5
    ((9, 4, 4, 4, 4, 4), 20000),     # order 6: the any-order instance
    ((1000, 10, 10, 10), 1),         # a single row
    ((50, 20, 20, 20), 2049),        # odd row count just past one span
])
def test_dense_kernel_edge_cases(oracle, shape, nnz):
    """Dense multi-vector kernel (keep = 0): short and long runs, span-crossing runs, orders
    2-6, odd and tiny row counts, gaps in the kept mode; within 1e-12 of the chained oracle."""
    import torch
    from paper_2510_01495_b200.device import DeviceCoo
    subs, vals = _canonical_coo(shape, nnz, seed=sum(shape) + nnz)
    t = DeviceCoo.from_host(subs, vals, shape)
    rng = np.random.default_rng(nnz)
    hv = {m: rng.random(shape[m]) + 0.5 for m in range(1, len(shape))}
    vecs = {m: torch.from_numpy(v).cuda() for m, v in hv.items()}
    out = t.ttv_dense(vecs, 0).cpu().numpy()
    ref = oracle.ttv_multi_dense(subs, vals, shape, hv, 0)
    assert np.array_equal(out != 0, ref != 0)
    nz = ref != 0
    assert np.max(np.abs(out[nz] - ref[nz]) / np.abs(ref[nz]), initial=0.0) <= REL
    # deterministic run to run
    assert t.ttv_dense(vecs, 0).cpu().numpy().tobytes() == out.tobytes()
    # 8-byte-aligned (not 16) columns: the scalar-load instance gives the same bits
    if t.nnz > 1:
        u = t.slice(1, t.nnz, copy=False)
        s1, v1 = subs[1:], vals[1:]
        o1 = u.ttv_dense(vecs, 0).cpu().numpy()
        r1 = oracle.ttv_multi_dense(s1, v1, shape, hv, 0)
        nz1 = r1 != 0
        assert np.array_equal(o1 != 0, nz1)
        assert np.max(np.abs(o1[nz1] - r1[nz1]) / np.abs(r1[nz1]), initial=0.0) <= REL


def test_dense_kernel_errors_and_unsorted(oracle):
    """Contracted index out of range raises DimensionError; an unsorted kept mode is detected
    and the chained path gives the (bit-exact) chained-oracle result."""
    import torch
    from paper_2510_01495_b200.device import DeviceCoo
    from paper_2510_01495_b200.errors import DimensionError
    shape = (30, 20, 20, 20)
    subs, vals = _canonical_coo(shape, 5000, seed=9)
    hv = {m: np.random.default_rng(m).random(shape[m]) + 0.5 for m in (1, 2, 3)}
    vecs = {m: torch.from_numpy(v).cuda() for m, v in hv.items()}
    bad = subs.copy()
    bad[1234, 2] = 20
    with pytest.raises(DimensionError):
        DeviceCoo.from_host(bad, vals, shape).ttv_dense(vecs, 0)
    perm = np.random.default_rng(3).permutation(len(vals))
    t = DeviceCoo.from_host(subs[perm], vals[perm], shape)
    out = t.ttv_dense(vecs, 0).cpu().numpy()
    ref = oracle.ttv_multi_dense(subs[perm], vals[perm], shape, hv, 0)
    assert out.tobytes() == ref.tobytes()


@pytest.mark.parametrize("shape,nnz,R,n", [
    ((200, 30, 40, 50), 60000, 16, 0),    # canonical n == 0: streams without a sort
    ((200, 30, 40, 50), 60000, 16, 2),    # other mode: device sort of the row ids
    ((5000, 3, 3, 3), 20000, 7, 0),       # runs of ~4 rows, rank not a multiple of 32
    ((1, 700, 800), 150000, 32, 0),       # one run over ~150 spans (carries + fix-up)
    ((60, 50), 2000, 40, 1),              # order 2, rank > 32 (two columns per lane)
    ((12, 5, 6, 7, 8, 3), 20000, 3, 0),   # order 6: the any-order instance
    ((40, 40, 40), 3001, 128, 1),         # rank 128 (four columns per lane)
    ((300, 40, 50), 200000, 3, 0),        # rank 3: eight rows per warp step, runs cross groups
    ((3000, 9, 9), 30000, 1, 0),          # rank 1 (the multi-vector TTV), short runs
    ((50, 20, 20, 20), 4099, 12, 3),      # last mode kept (sorted path), odd row count
])
def test_mttkrp_matches_chained_ttv_oracle(oracle, shape, nnz, R, n):
    """MTTKRP through the host C ABI and the device entry point: within
    1e-12 of the chained-TTV oracle, deterministic, zero rows for absent keys."""
    import torch
    import paper_2510_01495_b200 as tk
    from paper_2510_01495_b200.device import DeviceCoo
    subs, vals = _canonical_coo(shape, nnz, seed=nnz + R)
    rng = np.random.default_rng(R)
    U = [rng.random((s, R)) + 0.5 for s in shape]
    t = tk.SparseCooTensor(subs, vals, shape)
    got = tk.mttkrp(t, U, n)
    ref = oracle.mttkrp(subs, vals, shape, U, n) if R * nnz <= 2_000_000 else \
        oracle.mttkrp_fused(subs, vals, shape, U, n)
    nz = ref != 0
    assert np.array_equal(got != 0, nz)
    assert np.max(np.abs(got[nz] - ref[nz]) / ref[nz], initial=0.0) <= REL
    dt = DeviceCoo.from_host(subs, vals, shape)
    fac = {m: torch.from_numpy(U[m]).cuda() for m in range(len(shape)) if m != n}
    dev = dt.mttkrp(fac, n).cpu().numpy()
    assert dev.tobytes() == got.tobytes()
    assert dt.mttkrp(fac, n).cpu().numpy().tobytes() == dev.tobytes()


def test_mttkrp_errors_and_unsorted_input(oracle):
    import paper_2510_01495_b200 as tk
    from paper_2510_01495_b200.device import DeviceCoo
    from paper_2510_01495_b200.errors import DimensionError, ModeError
    import torch
    shape = (30, 20, 20)
    subs, vals = _canonical_coo(shape, 3000, seed=4)
    U = [np.random.default_rng(m).random((s, 4)) + 0.5 for m, s in enumerate(shape)]
    t = tk.SparseCooTensor(subs, vals, shape)
    with pytest.raises(ModeError):
        tk.mttkrp(t, U, 3)
    with pytest.raises(DimensionError):
        tk.mttkrp(t, [U[0], U[1][:10], U[2]], 0)
    bad = subs.copy()
    bad[100, 2] = 20
    fac = {m: torch.from_numpy(U[m]).cuda() for m in (1, 2)}
    with pytest.raises(DimensionError):
        DeviceCoo.from_host(bad, vals, shape).mttkrp(fac, 0)
    # rows out of kept-key order: detected, sorted on the device, same values as canonical
    perm = np.random.default_rng(2).permutation(len(vals))
    got = DeviceCoo.from_host(subs[perm], vals[perm], shape).mttkrp(fac, 0).cpu().numpy()
    ref = oracle.mttkrp(subs[perm], vals[perm], shape, U, 0)
    nz = ref != 0
    assert np.array_equal(got != 0, nz)
    assert np.max(np.abs(got[nz] - ref[nz]) / ref[nz]) <= REL


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_dense_peer_stores_merge_shards(oracle, world):
    """Sharded config-4-shaped dense TTV merged by the kernel's own stores
    (tk_ttv_dense_f64_device_peers): every shard writes its owned keep-mode range into all
    `world` output copies; afterwards every copy is identical, equals the chained oracle within
    1e-12, and carries exact zeros for keep indices without rows.  (One GPU, one process: the
    copies stand in for the peers' NVLink-mapped vectors; no kernel waits on another.)"""
    import torch
    from paper_2510_01495_b200 import multi
    from paper_2510_01495_b200.device import DeviceCoo
    shape = (3000, 40, 50, 60)
    subs, vals = _canonical_coo(shape, 400000, seed=31)
    keep_rows = subs[:, 0] % 7 != 3  # holes in the keep mode: owned indices without rows
    subs, vals = subs[keep_rows], vals[keep_rows]
    t = DeviceCoo.from_host(subs, vals, shape)
    hv = {m: np.random.default_rng(40 + m).random(shape[m]) + 0.5 for m in (1, 2, 3)}
    vecs = {m: torch.from_numpy(v).cuda() for m, v in hv.items()}
    ref = oracle.ttv_multi_dense(subs, vals, shape, hv, 0)
    outs = [torch.full((shape[0],), float("nan"), dtype=torch.float64, device="cuda") for _ in range(world)]
    key = t.cols[0]
    bounds = multi.shard_bounds(key, world)
    for r in range(world):
        lo, hi = multi.owned_key_range(key, bounds, r, shape[0])
        t.slice(bounds[r], bounds[r + 1]).ttv_dense_peers(vecs, 0, outs, lo, hi)
    torch.cuda.synchronize()
    got = [o.cpu().numpy() for o in outs]
    for g in got[1:]:
        assert g.tobytes() == got[0].tobytes()
    out = got[0]
    assert not np.isnan(out).any()
    assert np.array_equal(out == 0, ref == 0)
    nz = ref != 0
    assert np.max(np.abs(out[nz] - ref[nz]) / np.abs(ref[nz])) <= REL
    # an unsorted shard takes the chained path and still stores only its own range
    perm = np.random.default_rng(2).permutation(len(vals))
    u = DeviceCoo.from_host(subs[perm], vals[perm], shape)
    o2 = [torch.full((shape[0],), -1.0, dtype=torch.float64, device="cuda") for _ in range(2)]
    u.ttv_dense_peers(vecs, 0, o2, 100, 2000)
    for o in o2:
        h = o.cpu().numpy()
        assert (h[:100] == -1.0).all() and (h[2000:] == -1.0).all()
        assert h[100:2000].tobytes() == oracle.ttv_multi_dense(subs[perm], vals[perm], shape, hv, 0)[100:2000].tobytes()


def _ipc_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_01495_b200 import multi
        from paper_2510_01495_b200.device import DeviceCoo
        torch.cuda.set_device(0)
        shape = (500, 30, 30, 30)
        t = DeviceCoo.generate(shape, 300000, seed=77)
        vecs = {m: torch.rand(shape[m], dtype=torch.float64, device="cuda",
                              generator=torch.Generator(device="cuda").manual_seed(m)) for m in (1, 2, 3)}
        full = t.ttv_dense(vecs, 0).cpu().numpy()
        from gloo_comm import GlooComm
        merge = multi.PeerDenseMerge(shape[0], 0, GlooComm())
        bounds = multi.shard_bounds(t.cols[0], world)
        lo, hi = multi.owned_key_range(t.cols[0], bounds, rank, shape[0])
        out = merge.run(t.slice(bounds[rank], bounds[rank + 1]), vecs, 0, lo, hi).cpu().numpy()
        merge.close()
        rel = float(np.max(np.abs(out - full) / np.abs(full)))
        q.put((rank, rel, lo, hi))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc), -1, -1))
        raise
    finally:
        dist.destroy_process_group()


def test_dense_peer_merge_over_cuda_ipc_two_processes():
    """PeerDenseMerge end to end: two processes (both on cuda:0 -- one GPU here) export their
    output vectors by CUDA IPC, map each other's, and each shard's kernel stores its owned range
    into both; after the barrier both hold the full result (within 1e-12 of one-shot)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for rank, rel, lo, hi in res:
        assert not isinstance(rel, str), rel
        assert rel <= REL
    assert res[0][2] == 0 and res[0][3] == res[1][2] and res[1][3] == 500


def _split_case(queue, env):
    import os
    os.environ.update(env)
    from oracle import oracle
    from paper_2510_01495_b200 import backend
    K = backend.kernels()
    rng = np.random.default_rng(21)
    shape = (3000, 400, 900)
    n = 12_000_000
    cols = [np.minimum(rng.zipf(1.2, size=n) - 1, shape[0] - 1), rng.integers(0, shape[1], n),
            rng.integers(0, shape[2], n)]
    lin = np.unique(np.ravel_multi_index(cols, shape))
    subs = np.column_stack(np.unravel_index(lin, shape)).astype(np.int64)
    vals = rng.standard_normal(subs.shape[0])
    out = []
    for k in (1, 2):
        x = rng.standard_normal(shape[k])
        g, e = K.ttv_raw(subs, vals, shape, x, k), oracle.ttv_raw(subs, vals, shape, x, k)
        out.append(g[0].tobytes() == e[0].tobytes() and g[1].tobytes() == e[1].tobytes()
                   and tuple(g[2]) == tuple(e[2]))
    queue.put((subs.shape[0], out))


def _split_case4(queue, env):
    import os
    os.environ.update(env)
    from oracle import oracle
    from paper_2510_01495_b200 import backend
    K = backend.kernels()
    rng = np.random.default_rng(33)
    shape = (2000, 60, 50, 40)
    n = 9_000_000
    cols = [np.minimum(rng.zipf(1.1, size=n) - 1, shape[0] - 1)] + [rng.integers(0, m, n) for m in shape[1:]]
    lin = np.unique(np.ravel_multi_index(cols, shape))
    subs = np.column_stack(np.unravel_index(lin, shape)).astype(np.int64)
    vals = rng.standard_normal(subs.shape[0])
    out = []
    for k in (1, 2):
        x = rng.standard_normal(shape[k])
        g, e = K.ttv_raw(subs, vals, shape, x, k), oracle.ttv_raw(subs, vals, shape, x, k)
        out.append(g[0].tobytes() == e[0].tobytes() and g[1].tobytes() == e[1].tobytes())
    queue.put((subs.shape[0], out))


@pytest.mark.parametrize("env", [{"TK_SPLIT_MIN_NNZ": "1"},
                                 {"TK_SPLIT_MIN_NNZ": "1", "TK_SPLIT_MIN_ROWS": "100000"}])
def test_general_path_split_sort_order4(env):
    """Order-4 tensor, contracted mode 1 or 2 (R = product of two kept dims): the split path's
    part-local keys over three kept modes, one or many intervals; bit-exact against the oracle."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_split_case4, args=(q, env))
    pr.start()
    nrows, ok = q.get(timeout=600)
    pr.join(timeout=60)
    assert nrows > 3_000_000 and ok == [True, True], (env, nrows, ok)


@pytest.mark.parametrize("env", [
    {},                                                                     # one interval, 22-bit keys
    {"TK_SPLIT_MIN_ROWS": "150000"},                                        # many intervals, 2-3 passes
    {"TK_SPLIT_MIN_ROWS": "150000", "TK_SPLIT_MIN_NNZ": "1"},
    {"TK_SPLIT_SORT": "0"},                                                 # the one-sort path
])
def test_general_path_split_sort_bit_exact(env):
    """General path with the middle mode contracted on 6.9M canonical Zipf rows: the leading
    kept mode is sorted, so rows are cut into leading-mode intervals sorted on their own with
    32-bit keys.  Bit-exact against the oracle for k = 1 (and k = 2, the tile path), with one or
    many intervals (fresh process per setting: the switches are read once)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_split_case, args=(q, env))
    pr.start()
    nrows, ok = q.get(timeout=600)
    pr.join(timeout=60)
    assert nrows > 6_000_000 and ok == [True, True], (env, ok)


def _split_vs_one_sort(queue, env_off):
    import os
    if env_off:
        os.environ["TK_SPLIT_SORT"] = "0"
    import torch
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    t = DeviceCoo.generate((10**6, 10**5, 10**4), 50_000_000, zipf_s=1.2, normal_vals=True, seed=12345)
    x = uniform_vector(10**5, 778)
    u, s, v = t.ttv(x, 1)
    queue.put((u, hashlib.sha256(s[:u].cpu().numpy().tobytes()).hexdigest(),
               hashlib.sha256(v[:u].cpu().numpy().tobytes()).hexdigest()))


def test_general_path_split_matches_one_sort_at_scale():
    """Config-5 tensor shape (Zipf 1.2, 5e7 rows), middle mode: the split path and the one-sort
    path (TK_SPLIT_SORT=0, fresh process) give the same bytes."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    res = []
    for off in (False, True):
        q = ctx.Queue()
        pr = ctx.Process(target=_split_vs_one_sort, args=(q, off))
        pr.start()
        res.append(q.get(timeout=600))
        pr.join(timeout=60)
    assert res[0] == res[1]


def test_c_abi_timed_and_one_process_multi_device(oracle):
    """The timed device entry points (event pair around the call) and tk_multi_ttv_f64: three
    key-aligned shards, all on device 0 here (one host thread per shard), concatenate to the
    one-call result bit for bit; offsets are the exclusive prefix of the shard counts."""
    import ctypes
    import torch
    from paper_2510_01495_b200 import _lib, multi
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    lib = _lib.load()
    shape = (2000, 300, 400)
    t = DeviceCoo.generate(shape, 3_000_000, zipf_s=1.1, normal_vals=True, seed=5)
    x = uniform_vector(shape[2], 9)
    u0, s0, v0 = t.ttv(x, 2)
    ms = ctypes.c_float(-1.0)
    os_ = torch.empty((t.nnz, 2), dtype=torch.int64, device="cuda")
    ov = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
    u = ctypes.c_int64(0)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.tk_ttv_f64_device_timed(3, _lib.i64_array(shape), t.nnz,
                                           _lib.ptr_array([c.data_ptr() for c in t.cols]), None, t.vals.data_ptr(),
                                           x.data_ptr(), shape[2], 2, os_.data_ptr(), ov.data_ptr(), ctypes.byref(u),
                                           st, ctypes.byref(ms)))
    assert u.value == u0 and ms.value > 0
    assert torch.equal(os_[:u0], s0[:u0]) and torch.equal(ov[:u0], v0[:u0])
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.check(lib.tk_dot_f64_device_timed(t.vals.data_ptr(), t.vals.data_ptr(), t.nnz, out.data_ptr(), st,
                                           ctypes.byref(ms)))
    assert ms.value > 0
    # one process, three shards on device 0
    key = multi.kept_prefix_key(t.cols, 2, shape)
    bounds = multi.shard_bounds(key, 3)
    shards = [t.slice(bounds[i], bounds[i + 1]) for i in range(3)]
    outs = [(torch.empty((max(sh.nnz, 1), 2), dtype=torch.int64, device="cuda"),
             torch.empty(max(sh.nnz, 1), dtype=torch.float64, device="cuda")) for sh in shards]
    dev = (ctypes.c_int32 * 3)(0, 0, 0)
    _lib.check(lib.tk_multi_init(1, (ctypes.c_int32 * 1)(0)))
    col_arrays = [_lib.ptr_array([c.data_ptr() for c in sh.cols]) for sh in shards]
    cols_pp = (ctypes.c_void_p * 3)(*[ctypes.cast(a, ctypes.c_void_p).value for a in col_arrays])
    nnz = (ctypes.c_int64 * 3)(*[sh.nnz for sh in shards])
    counts, offs = (ctypes.c_int64 * 3)(), (ctypes.c_int64 * 4)()
    _lib.check(lib.tk_multi_ttv_f64(3, _lib.i64_array(shape), 2, 3, dev, nnz, cols_pp,
                                    _lib.ptr_array([sh.vals.data_ptr() for sh in shards]),
                                    _lib.ptr_array([x.data_ptr()] * 3), shape[2],
                                    _lib.ptr_array([o[0].data_ptr() for o in outs]),
                                    _lib.ptr_array([o[1].data_ptr() for o in outs]), counts, offs))
    _lib.check(lib.tk_multi_free())
    assert list(offs) == [0, counts[0], counts[0] + counts[1], u0]
    cat_s = torch.cat([outs[i][0][:counts[i]] for i in range(3)])
    cat_v = torch.cat([outs[i][1][:counts[i]] for i in range(3)])
    assert torch.equal(cat_s, s0[:u0]) and torch.equal(cat_v, v0[:u0])


def test_cfg5_shape_1e8_rows_against_reference(oracle):
    """Full-scale parity: 1e8 rows of the config-5 shape (Zipf 1.2, N(0,1)
    values), the device TTV and the drop-in host call (pageable arrays, packed staging) against the
    reference's own kernel (oracle/_ref, key-aligned shards on every host thread) -- bit-exact."""
    import paper_2510_01495_b200 as tk
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    shape = (10**6, 10**5, 10**4)
    t = DeviceCoo.generate(shape, 100_000_000, zipf_s=1.2, normal_vals=True, seed=12345)
    x = uniform_vector(shape[2], 777)
    u, os_d, ov_d = t.ttv(x, 2)
    gs, gv = os_d[:u].cpu().numpy(), ov_d[:u].cpu().numpy()
    subs, vals = t.to_host()
    del t, os_d, ov_d
    xh = x.cpu().numpy()
    parts, _, kind = oracle.ttv_raw_threads(subs, vals, shape, xh, 2)
    assert oracle.compare_parts(parts, gs, gv), kind
    hs, hv, hsh = tk.kernels().ttv_raw(subs, vals, shape, xh, 2)
    assert hsh == (shape[0], shape[1])
    assert oracle.compare_parts(parts, hs, hv)


def test_cfg4_shape_1e8_rows_against_chained_reference(oracle):
    """Config 4 at full size: the fused dense TTV within 1e-12 relative of the chain of the
    reference's ttv_raw (modes 3, 2, 1), densified -- SURVEY 8c's config-4 oracle."""
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    shape = (20000,) * 4
    t = DeviceCoo.generate(shape, 100_000_000, seed=4444)
    vecs = {m: uniform_vector(shape[m], 40 + m) for m in (1, 2, 3)}
    got = t.ttv_dense(vecs, 0).cpu().numpy()
    subs, vals = t.to_host()
    del t
    ref, _, _ = oracle.ttv_multi_dense_threads(subs, vals, shape, {m: v.cpu().numpy() for m, v in vecs.items()}, 0)
    nz = ref != 0
    assert np.array_equal(got[~nz], ref[~nz])
    assert np.max(np.abs(got[nz] - ref[nz]) / np.abs(ref[nz])) <= 1e-12


def test_tile_three_pass_fallback_bit_exact(oracle, monkeypatch, golden_small, golden_hashes):
    """The order-independent fallback of the single-pass tile kernel (count pass, one-CTA scan,
    fold pass -- what a call re-runs if in-order block dispatch ever fails and a wait gives up),
    forced with TK_TILE_MULTIPASS=1: bit-exact on the golden cases and on a Zipf tensor with
    groups spanning many tiles, sorted-stream and sort paths."""
    import paper_2510_01495_b200 as tk
    monkeypatch.setenv("TK_TILE_MULTIPASS", "1")
    K = tk.kernels()
    n = 0
    for name, subs, vals, shape, x, k, err, exp in ttv_cases(golden_small, golden_hashes):
        if err:
            continue
        s, v, sh = K.ttv_raw(subs, vals, shape, x, k)
        assert s.tobytes() == exp[0].tobytes() and v.tobytes() == exp[1].tobytes(), name
        n += 1
    assert n >= 100
    shape = (2000, 300, 400)
    subs, vals = oracle.gen_coo(shape, 3_000_000, zipf_s=1.3, normal_vals=True, seed=8)
    for k in (2, 1, 0):
        x = oracle.gen_uniform(shape[k], 3 + k)
        es, ev, _ = oracle.ttv_raw(subs, vals, shape, x, k)
        s, v, _ = K.ttv_raw(subs, vals, shape, x, k)
        assert s.tobytes() == es.tobytes() and v.tobytes() == ev.tobytes(), k


def test_tile_kernel_beside_concurrent_kernels(oracle):
    """The single-pass tile kernel relies on its blocks being dispatched in index order while it
    shares the GPU: with another stream keeping every SM busy (back-to-back GEMMs and copies) the
    device-resident TTV -- sorted-stream path and the middle-mode path -- is still bit-exact
    against the oracle, call after call (a stalled wait would re-run the call as three passes or
    fail it; either way the result must be right)."""
    import torch
    from paper_2510_01495_b200.device import DeviceCoo
    shape = (3000, 500, 600)
    subs, vals = oracle.gen_coo(shape, 6_000_000, zipf_s=1.2, normal_vals=True, seed=31)
    t = DeviceCoo.from_host(subs, vals, shape)
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    big = torch.empty(64 * 2**20, device="cuda", dtype=torch.float32)
    for k in (2, 1):
        x_h = oracle.gen_uniform(shape[k], 40 + k)
        es, ev, _ = oracle.ttv_raw(subs, vals, shape, x_h, k)
        x = torch.from_numpy(x_h).cuda()
        torch.cuda.synchronize()
        for rep in range(4):
            with torch.cuda.stream(side):  # ~20 ms of work on the other stream, queued first
                for _ in range(12):
                    b = a @ a
                    big.add_(1.0)
            u, os_d, ov_d = t.ttv(x, k)
            gs, gv = os_d[:u].cpu().numpy(), ov_d[:u].cpu().numpy()
            assert gs.tobytes() == es.tobytes() and gv.tobytes() == ev.tobytes(), (k, rep)
        torch.cuda.synchronize()


def test_nccl_comm_inside_the_library_single_rank():
    """The C-ABI NCCL data plane (tk_nccl_*) on the one GPU of the test box: a one-rank
    communicator runs every exchange the sharded TTV uses -- the count all-gather (pipelined
    tickets), the gather of sparse slices to the root, the IPC-handle exchange, the stream-ordered
    barrier and the all-reduce merge -- and the peer-store dense merge driven through it."""
    import torch
    from paper_2510_01495_b200 import multi
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    comm = multi.NcclComm(0, 1, bootstrap=lambda uid: uid)
    try:
        t1, t2 = comm.counts_start(7), comm.counts_start(9)
        assert comm.counts_wait(t1) == [7] and comm.counts_wait(t2) == [9]
        s = torch.arange(10, dtype=torch.int64, device="cuda").reshape(5, 2)
        v = torch.rand(5, dtype=torch.float64, device="cuda")
        gs, gv = multi.gather_sparse_to_root(comm, s, v, [5])
        assert torch.equal(gs, s) and torch.equal(gv, v)
        assert comm.allgather_bytes(b"h" * 64) == [b"h" * 64]
        x = torch.rand(1000, dtype=torch.float64, device="cuda")
        y = x.clone()
        multi.merge_dense(comm, y)
        comm.barrier()
        torch.cuda.synchronize()
        assert torch.equal(x, y)
        shape = (500, 30, 30, 30)
        t = DeviceCoo.generate(shape, 200000, seed=12)
        vecs = {m: uniform_vector(shape[m], 60 + m) for m in (1, 2, 3)}
        full = t.ttv_dense(vecs, 0)
        merge = multi.PeerDenseMerge(shape[0], torch.cuda.current_device(), comm)
        out = merge.run(t, vecs, 0, 0, shape[0])
        torch.cuda.synchronize()
        assert torch.equal(out, full)
        merge.close()
    finally:
        comm.close()


@pytest.mark.parametrize("shape,nnz,zipf,env", [
    ((400, 300, 200), 600_000, 1.3, {}),                             # Zipf: classes A, M and B at once
    ((50, 300, 200), 2_000_000, 1.2, {}),                            # class B + M segments
    ((20, 200, 200), 500_000, 0.0, {}),                              # class M only (25K-row segments)
    ((60, 80, 90), 200_000, 1.1, {"TK_MID_TILE": "97", "TK_MID_MEDMAX": "2048"}),  # many B tiles + chunks
    ((30, 40, 20, 10), 150_000, 1.2, {"TK_MID_TILE": "257", "TK_MID_MEDMAX": "2048"}),  # order 4
    ((30, 40, 20, 10), 150_000, 1.2, {}),                            # order 4, class M
    ((3000, 20, 30), 400_000, 0.0, {}),                              # class A only
    ((200000, 50, 40), 300_000, 0.0, {}),                            # tiny segments, empty leading values
    ((40, 3000, 2), 200_000, 1.1, {}),                               # R = 2: one or two owner warps, long single-S chains
    ((6, 200000, 1), 900_000, 0.0, {"TK_MID_MEDMAX": "4096"}),       # R = 1: every row one S (classes M and B, 150K-row chains)
    ((30, 50, 16384), 300_000, 0.0, {}),                             # R = 2^14: the widest accumulator array
    ((700, 40, 600), 700_000, 0.9, {}),                              # segments around the class A / M boundary (512 rows)
])
def test_middle_mode_counting_path_bit_exact(oracle, monkeypatch, shape, nnz, zipf, env):
    """k == 1 (the paper's middle-mode protocol) through the segmented counting path
    (tk_midmode.cu): class-A warp-per-segment accumulation, class-M owner lists with in-place
    accumulators, class-B counting tiles, owner-list scatter and the binned bucket folds --
    bit-exact against the oracle, with the class thresholds shrunk to put small data through every
    class and many tiles."""
    import paper_2510_01495_b200 as tk
    for kk, vv in env.items():
        monkeypatch.setenv(kk, vv)
    s, v = oracle.gen_coo(shape, nnz, zipf_s=zipf, normal_vals=True, seed=17)
    x = oracle.gen_uniform(shape[1], 5)
    es, ev, _ = oracle.ttv_raw(s, v, shape, x, 1)
    gs, gv, gsh = tk.kernels().ttv_raw(s, v, shape, x, 1)
    assert gs.tobytes() == es.tobytes() and gv.tobytes() == ev.tobytes() and len(ev) > 0


def test_middle_mode_exact_class_boundaries(oracle):
    """Segments of exactly 1, 2, 31, 32, 33, 511, 512, 513, 1023, 1024, 1025, 65535, 65536 and
    65537 rows (the class A / M / B thresholds and the 32-row step and 1024-row chunk edges), with
    empty leading values in between -- bit-exact against the oracle."""
    import paper_2510_01495_b200 as tk
    rng = np.random.default_rng(23)
    n1, n2 = 300, 300
    sizes = [1, 0, 2, 31, 32, 33, 0, 0, 511, 512, 513, 1023, 1024, 1025, 65535, 65536, 65537, 0, 7]
    rows = []
    for i0, L in enumerate(sizes):
        flat = np.sort(rng.choice(n1 * n2, size=L, replace=False))
        rows.append(np.stack([np.full(L, i0), flat // n2, flat % n2], axis=1))
    s = np.concatenate(rows).astype(np.int64)
    v = rng.standard_normal(len(s))
    shape = (len(sizes), n1, n2)
    x = oracle.gen_uniform(n1, 9)
    es, ev, _ = oracle.ttv_raw(s, v, shape, x, 1)
    gs, gv, _ = tk.kernels().ttv_raw(s, v, shape, x, 1)
    assert gs.tobytes() == es.tobytes() and gv.tobytes() == ev.tobytes() and len(ev) > 0


def test_middle_mode_zero_groups_errors_and_declines(oracle):
    """Exact-zero groups are removed (compaction), an out-of-range contracted index raises
    DimensionError, garbage kept indices and an unsorted leading column decline to the general
    paths -- all matching the oracle."""
    import paper_2510_01495_b200 as tk
    from paper_2510_01495_b200 import errors
    K = tk.kernels()
    shape = (20, 50, 30)
    s, v = oracle.gen_coo(shape, 20000, seed=3)
    v = v.copy()
    # cancelling pairs: rows with equal (i0, i2) and adjacent i1 get +a / -a
    key = s[:, 0] * 10**6 + s[:, 2]
    order = np.lexsort((s[:, 1], key))
    for a, b in zip(order[:-1:2], order[1::2]):
        if key[a] == key[b] and a % 3 == 0:
            v[b] = -v[a]
    x = np.ones(shape[1])
    es, ev, _ = oracle.ttv_raw(s, v, shape, x, 1)
    gs, gv, _ = K.ttv_raw(s, v, shape, x, 1)
    assert gs.tobytes() == es.tobytes() and gv.tobytes() == ev.tobytes()
    bad = s.copy()
    bad[777, 1] = shape[1]
    with pytest.raises(errors.DimensionError):
        K.ttv_raw(bad, v, shape, x, 1)
    g = s.copy()
    g[5, 2] = -3  # garbage kept index
    es, ev, _ = oracle.ttv_raw(g, v, shape, x, 1)
    gs, gv, _ = K.ttv_raw(g, v, shape, x, 1)
    assert gs.tobytes() == es.tobytes() and gv.tobytes() == ev.tobytes()
    perm = np.random.default_rng(1).permutation(len(v))  # leading column unsorted
    es, ev, _ = oracle.ttv_raw(s[perm], v[perm], shape, x, 1)
    gs, gv, _ = K.ttv_raw(s[perm], v[perm], shape, x, 1)
    assert gs.tobytes() == es.tobytes() and gv.tobytes() == ev.tobytes()


def test_cfg5_shape_middle_mode_1e8_rows_against_reference(oracle):
    """The paper's protocol at scale: config-5 shape, 1e8 rows, k = 1 (contract the middle mode)
    -- the counting path against the reference's own kernel on every host thread (shards cut at
    leading-value changes), bit-exact."""
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    shape = (10**6, 10**5, 10**4)
    t = DeviceCoo.generate(shape, 100_000_000, zipf_s=1.2, normal_vals=True, seed=12345)
    x = uniform_vector(shape[1], 778)
    u, os_d, ov_d = t.ttv(x, 1)
    gs, gv = os_d[:u].cpu().numpy(), ov_d[:u].cpu().numpy()
    subs, vals = t.to_host()
    del t, os_d, ov_d
    parts, _, kind = oracle.ttv_raw_threads(subs, vals, shape, x.cpu().numpy(), 1)
    assert oracle.compare_parts(parts, gs, gv), kind
