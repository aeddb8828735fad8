"""The B200 module driven through the reference's own harness: its implementation registry
(tenkern.bench ImplEntry / run_experiment, bench.py:191-215, 387-431), the host toolbox's
BoundKernelSet (tenhost/bindings.py:40-79) and its first-call overhead estimator
(tenhost/overhead.py:76-175).  The reference packages are the ones oracle/Makefile stages into
oracle/_ref (test infrastructure); the tests skip when that staging is absent."""

import os
import sys

import numpy as np
import pytest

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "tenhost")):
        pytest.skip("reference packages not staged (make -C oracle ref)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import tenkern
    import tenhost  # noqa: F401
    from paper_2510_01495_b200 import registry
    registry.register()
    return tenkern


def test_labels_registered(ref):
    impls = ref.implementations()
    assert {"b200", "b200-via-ffi", "native-loop", "host-vectorized"} <= set(impls)
    e = impls["b200"]
    assert e.self_timed and e.experiments == ref.EXPERIMENTS
    assert not impls["b200-via-ffi"].self_timed


def test_unavailable_without_gpu(ref):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    assert not ref.implementations()["b200"].available()
    cfg = ref.ExperimentConfig("dot", sizes=(100,), n_trials=1)
    with pytest.raises(ref.ConfigError, match="b200"):
        ref.run_experiment(cfg, ["b200"])
    from paper_2510_01495_b200 import registry
    with pytest.raises(ref.ConfigError):  # the reference's own label check, before any child
        registry.estimate_overhead(1000, experiment="dot", repeats=1)


def _thunk_out(ref, label, cfg, size):
    from tenkern.bench import build_operands, derive_trial_seed
    entry = ref.implementations()[label]
    data = build_operands(cfg, size, derive_trial_seed(cfg.seed, 0, 0))
    out = entry.make_thunk(cfg.experiment, data, cfg.checked)()
    return out[0] if entry.self_timed else out


@pytest.mark.gpu
@pytest.mark.parametrize("experiment,size,extra", [
    ("dot", 1_000_000, {}),
    ("matvec_square", 512, {}),
    ("matvec_rows", 10_000, {}),
    ("ttv", 200, {"density": 0.01, "mode": 2}),
    ("ttv", 300, {"density": 0.001, "mode": 3}),
    ("ttv", 100, {"density": 0.05, "mode": 1}),
])
def test_b200_label_matches_native_loop(ref, experiment, size, extra):
    cfg = ref.ExperimentConfig(experiment, sizes=(size,), n_trials=2, **extra)
    for label in ("b200", "b200-via-ffi"):
        got = _thunk_out(ref, label, cfg, size)
        exp = _thunk_out(ref, "native-loop", cfg, size)
        if experiment == "ttv":
            gs, gv = (got.subs, got.vals) if hasattr(got, "subs") else (got[0], got[1])  # HostSparseTensor
            es, ev = exp[0], exp[1]
            assert np.asarray(gs).tobytes() == np.asarray(es).tobytes(), label
            assert np.asarray(gv).tobytes() == np.asarray(ev).tobytes(), label
        else:
            np.testing.assert_allclose(got, exp, rtol=1e-12, atol=0)
    recs = ref.run_experiment(cfg, ["b200", "native-loop"])
    summ = ref.summarize(recs)
    assert [s.implementation for s in summ] == ["b200", "native-loop"]
    assert all(s.n == 2 and s.mean_s > 0 for s in summ)


@pytest.mark.gpu
def test_bound_kernel_set_with_b200_module(ref):
    from tenhost.bindings import BoundKernelSet, bound_kernels
    import paper_2510_01495_b200 as tk
    ours, theirs = BoundKernelSet(kernel_module=tk.kernels()), bound_kernels()
    r = np.random.default_rng(3)
    a, x = r.random((300, 200)), r.random(200)
    np.testing.assert_allclose(ours.matvec(a, x), theirs.matvec(a, x), rtol=1e-12, atol=0)
    assert ours.dot(x, x) == pytest.approx(theirs.dot(x, x), rel=1e-12)
    t = ref.gen_sparse3(ref.GenSpec(9, "sparse3", (80, 70, 60), 0.02))
    v = r.random(70)
    got, exp = ours.ttv(t.subs, t.vals, t.shape, v, 1), theirs.ttv(t.subs, t.vals, t.shape, v, 1)
    assert got.new_subs.tobytes() == exp.new_subs.tobytes() and got.new_vals.tobytes() == exp.new_vals.tobytes()
    assert got.new_shape == exp.new_shape


@pytest.mark.gpu
def test_first_call_overhead_through_reference_estimator(ref):
    from paper_2510_01495_b200 import registry
    est = registry.estimate_overhead(100_000, experiment="dot", n_trials=5, repeats=2, timeout_s=300)
    assert est.kernel == "b200" and est.repeats == 2
    assert est.first_call_mean_s > est.steady_mean_s > 0
    est = registry.estimate_overhead(100, experiment="ttv", n_trials=3, repeats=2, timeout_s=300)
    assert est.repeats == 2 and est.overhead_s > 0
