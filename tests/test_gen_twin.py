"""The host twin of the operand generator (oracle/tk_gen_host.cpp) against its contract and,
on the GPU, against the device generator (csrc/tk_gen.cu) byte for byte.

The bench's reference arm builds the config-4/5 tensors with the host twin (it must not load the
product library), so "same_config" rests on these checks."""

import numpy as np
import pytest


def _canonical_distinct(subs):
    if subs.shape[0] < 2:
        return True
    d = np.diff(subs, axis=0)
    # first non-zero column of every row difference must be positive
    nz = d != 0
    first = np.argmax(nz, axis=1)
    return bool(np.all(nz.any(axis=1)) and np.all(d[np.arange(d.shape[0]), first] > 0))


@pytest.mark.parametrize("shape,nnz,zipf,normal", [
    ((50, 40, 30), 5000, 0.0, False),
    ((1000, 100, 10), 20000, 1.2, True),
    ((20, 20, 20, 20), 30000, 0.0, False),
    ((7, 5), 35, 0.0, True),  # every cell
])
def test_host_generator_contract(oracle, shape, nnz, zipf, normal):
    s, v = oracle.gen_coo(shape, nnz, zipf_s=zipf, normal_vals=normal, seed=11, threads=3)
    assert s.shape == (nnz, len(shape)) and v.shape == (nnz,)
    assert _canonical_distinct(s)
    assert np.all(s >= 0) and np.all(s < np.asarray(shape))
    assert np.all(v != 0.0)
    if not normal:
        assert np.all((v > 0) & (v < 1))
    # deterministic and independent of the thread count
    s2, v2 = oracle.gen_coo(shape, nnz, zipf_s=zipf, normal_vals=normal, seed=11, threads=1)
    assert s.tobytes() == s2.tobytes() and v.tobytes() == v2.tobytes()


def test_host_generator_first_distinct_semantics(oracle):
    """Growing nnz only appends draws: the nnz-tensor is a subset of the (nnz+k)-tensor (the
    first-nnz-distinct-draws protocol of synth.py:124-131)."""
    shape = (30, 30, 30)
    a, _ = oracle.gen_coo(shape, 2000, zipf_s=1.1, seed=5)
    b, _ = oracle.gen_coo(shape, 2600, zipf_s=1.1, seed=5)
    ka = {tuple(r) for r in a}
    kb = {tuple(r) for r in b}
    assert ka <= kb and len(kb) == 2600


def test_exact_op_normal_transform(oracle):
    """ln / cos made of exactly rounded operations are accurate (the values are a real N(0,1))."""
    import math
    L = oracle.gen_lib()
    r = np.random.default_rng(0)
    for x in list(r.random(2000)) + [1.0, 2.0**-53, 0.5]:
        if x > 0:
            assert abs(L.tkg_ln(x) - math.log(x)) <= 4e-16 * max(1.0, abs(math.log(x)))
    for t in r.random(2000):
        assert abs(L.tkg_cos2pi(t) - math.cos(2 * math.pi * t)) <= 1e-15
    _, v = oracle.gen_coo((100, 100, 100), 200000, normal_vals=True, seed=3)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1.0) < 0.01


@pytest.mark.gpu
@pytest.mark.parametrize("shape,nnz,zipf,normal,seed", [
    ((50, 40, 30), 5000, 0.0, False, 1),
    ((1000, 1000, 1000), 1_000_000, 0.0, False, 2),
    ((10**6, 10**5, 10**4), 3_000_000, 1.2, True, 12345),
    ((20000,) * 4, 2_000_000, 0.0, False, 4444),
    ((300, 200, 100), 400000, 1.1, True, 9),
])
def test_device_generator_matches_host_twin(oracle, shape, nnz, zipf, normal, seed):
    import torch
    from paper_2510_01495_b200.device import DeviceCoo
    t = DeviceCoo.generate(shape, nnz, zipf_s=zipf, normal_vals=normal, seed=seed)
    ds, dv = t.to_host()
    hs, hv = oracle.gen_coo(shape, nnz, zipf_s=zipf, normal_vals=normal, seed=seed)
    assert ds.tobytes() == hs.tobytes()
    assert dv.tobytes() == hv.tobytes()
    del t
    torch.cuda.empty_cache()


@pytest.mark.gpu
def test_device_uniform_vector_matches_host_twin(oracle):
    from paper_2510_01495_b200.device import uniform_vector
    for n, seed in ((1, 3), (1000, 777), (100003, 2**40 + 5)):
        assert uniform_vector(n, seed).cpu().numpy().tobytes() == oracle.gen_uniform(n, seed).tobytes()
