"""Host-side logic that needs no GPU: API surface, canonical form, errors, generators."""

import numpy as np
import pytest

import paper_2510_01495_b200 as tk
from paper_2510_01495_b200 import backend, errors, sparse, synth


def test_public_surface_mirrors_reference():
    for name in ("dot", "matvec", "ttv", "SparseCooTensor", "TtvRawResult", "densify", "set_difference",
                 "unique_rows_accumulate", "as_vector", "as_matrix", "kernels", "active_backend",
                 "DimensionError", "ModeError", "OrderError", "SizeCapError", "GenSpec", "gen_sparse3"):
        assert hasattr(tk, name), name


def test_kernel_module_protocol():
    k = backend.kernels()
    assert k.BACKEND == "b200" and k.SELF_TIMED is True
    for fn in ("dot", "matvec", "ttv_raw", "dot_timed", "matvec_timed", "ttv_timed"):
        assert callable(getattr(k, fn))
    assert backend.kernels("b200") is k
    with pytest.raises(errors.ConfigError):
        backend.kernels("compiled")
    with pytest.raises(errors.ConfigError):
        backend.kernels("fortran")


def test_canonical_input_taken_as_is_without_device():
    rng = np.random.default_rng(1)
    vals = rng.random(3) + 0.5
    t = tk.SparseCooTensor([[0, 0], [0, 1], [1, 0]], vals, (2, 2))
    assert t.vals.tobytes() == vals.tobytes()
    with pytest.raises(ValueError):
        t.vals[0] = 2.0
    with pytest.raises(AttributeError):
        t.shape = (3, 3)


def test_construction_errors():
    with pytest.raises(errors.DimensionError):
        tk.SparseCooTensor([[2, 0]], [1.0], (2, 2))
    with pytest.raises(errors.DimensionError):
        tk.SparseCooTensor([[-1, 0]], [1.0], (2, 2))
    with pytest.raises(errors.DimensionError):
        tk.SparseCooTensor([[0, 0]], [1.0, 2.0], (2, 2))
    with pytest.raises(errors.DimensionError):
        tk.SparseCooTensor([[0, 0]], [1.0], (2, 0))
    with pytest.raises(errors.OrderError):
        tk.SparseCooTensor(np.empty((0, 0)), [], ())


def test_equality_repr_densify_roundtrip():
    a = tk.SparseCooTensor([[0, 1]], [5.0], (2, 2))
    assert a == tk.SparseCooTensor([[0, 1]], [5.0], (2, 2))
    assert a != tk.SparseCooTensor([[0, 1]], [5.0], (2, 3)) and a != "x"
    assert "(2, 2)" in repr(a)
    assert np.array_equal(tk.densify(a), [[0.0, 5.0], [0.0, 0.0]])
    assert tk.SparseCooTensor.from_dense(tk.densify(a)) == a
    with pytest.raises(errors.SizeCapError):
        tk.densify(tk.SparseCooTensor([[0, 0, 0]], [1.0], (101, 101, 101)))


def test_set_difference():
    assert tk.set_difference([0, 1, 2], [1]) == [0, 2]
    assert tk.set_difference([0, 1, 2, 3], []) == [0, 1, 2, 3]
    assert tk.set_difference([0, 5, 9], [7, 100]) == [0, 5, 9]


def test_ttv_argument_errors_without_device():
    t = tk.SparseCooTensor([[0, 0, 0]], [1.0], (3, 4, 5))
    with pytest.raises(errors.ModeError):
        tk.ttv(t, np.ones(3), 3)
    with pytest.raises(errors.ModeError):
        tk.ttv(t, np.ones(3), -1)
    with pytest.raises(errors.DimensionError):
        tk.ttv(t, np.ones(4), 0)
    with pytest.raises(errors.OrderError):
        tk.ttv(tk.SparseCooTensor([[1]], [2.0], (4,)), np.ones(4), 0)


def test_dense_coercion_errors():
    with pytest.raises(errors.DimensionError):
        tk.dot([[1.0]], [[1.0]])
    with pytest.raises(errors.DimensionError):
        tk.matvec([1.0, 2.0], [1.0])
    with pytest.raises(errors.DimensionError) as e:
        tk.dot([1.0, 2.0], [1.0, 2.0, 3.0])
    assert "2" in str(e.value) and "3" in str(e.value)


def test_gen_sparse3_exact_density_protocol():
    t = synth.gen_sparse3(synth.GenSpec(424242, "sparse3", (100, 100, 100), 0.01))
    assert t.nnz == 10000
    assert (t.vals > 0.0).all() and (t.vals < 1.0).all()
    assert sparse._rows_strictly_increasing(t.subs)


def test_genspec_validation():
    with pytest.raises(errors.GenerationError):
        synth.GenSpec(1, "tensor", (3,))
    with pytest.raises(errors.GenerationError):
        synth.GenSpec(1, "sparse3", (3, 3, 3))
    with pytest.raises(errors.GenerationError):
        synth.GenSpec(1, "sparse3", (3, 3, 3), 1e-9)
    with pytest.raises(errors.GenerationError):
        synth.GenSpec(-1, "vector", (3,))
