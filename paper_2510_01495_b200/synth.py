"""Seeded operands for the BASELINE configurations.

Configs 1-3 are generated on the host exactly as the reference's harness does, so the
bytes are identical to what the reference's own ``bench.build_operands`` hands its
kernels (pinned by tests/golden/golden_hashes.json):

* PCG64 ``numpy.random.default_rng`` (synth.py:23), per-batch seeds from
  ``SeedSequence((master, size_index, schedule_index))`` and per-argument seeds from
  ``SeedSequence((trial_seed, arg_index))`` (bench.py:349-363);
* vectors / matrices i.i.d. uniform [0,1) (synth.py:89-100);
* order-3 tensors with an exact nonzero count: draw linear indices, dedupe, top up until
  exactly nnz, values uniform with zeros redrawn, indices drawn before values
  (synth.py:103-143).

Configs 4 and 5 (1e8 / 4e8 nonzeros) are generated on the device by ``tk_gen_coo_device``
(see csrc/tk_gen.cu) with the same exact-nnz semantics; ``device.DeviceCoo.generate``.
"""

from dataclasses import dataclass

import numpy as np

from .errors import GenerationError
from .sparse import SparseCooTensor

__all__ = ["GENERATOR", "GenSpec", "gen_vector", "gen_matrix", "gen_sparse3",
           "derive_trial_seed", "derive_arg_seed", "CONFIGS", "host_operands"]

GENERATOR = "numpy.random.default_rng(PCG64)"
DEFAULT_SEED = 12345  # reference default master seed, bench.py:66

_ORDER = {"vector": 1, "matrix": 2, "sparse3": 3}


@dataclass(frozen=True)
class GenSpec:
    """Recipe for one generated operand (synth.py:30-86)."""

    seed: int
    kind: str
    dims: tuple
    density: float = None

    def __post_init__(self):
        if self.kind not in _ORDER:
            raise GenerationError(f"unknown kind {self.kind!r}")
        seed = int(self.seed)
        if not 0 <= seed < 2**64:
            raise GenerationError(f"seed must be an unsigned 64-bit int, got {seed}")
        object.__setattr__(self, "seed", seed)
        dims = tuple(int(n) for n in self.dims)
        if len(dims) != _ORDER[self.kind]:
            raise GenerationError(f"kind {self.kind!r} needs {_ORDER[self.kind]} dims, got {dims}")
        if any(n <= 0 for n in dims):
            raise GenerationError(f"dims entries must be positive, got {dims}")
        object.__setattr__(self, "dims", dims)
        if self.kind == "sparse3":
            if self.density is None:
                raise GenerationError("sparse3 spec needs a density")
            density = float(self.density)
            if not 0.0 < density <= 1.0:
                raise GenerationError(f"density must lie in (0, 1], got {density}")
            if density * int(np.prod(dims, dtype=object)) < 1.0:
                raise GenerationError(f"degenerate spec: density {density} yields no nonzeros")
            object.__setattr__(self, "density", density)
        elif self.density is not None:
            raise GenerationError(f"kind {self.kind!r} takes no density")

    @property
    def nnz(self) -> int:
        if self.kind != "sparse3":
            raise GenerationError(f"kind {self.kind!r} has no nnz")
        return int(round(self.density * int(np.prod(self.dims, dtype=object))))


def gen_vector(spec: GenSpec) -> np.ndarray:
    if spec.kind != "vector":
        raise GenerationError(f"gen_vector got a {spec.kind!r} spec")
    return np.random.default_rng(spec.seed).random(spec.dims[0])


def gen_matrix(spec: GenSpec) -> np.ndarray:
    if spec.kind != "matrix":
        raise GenerationError(f"gen_matrix got a {spec.kind!r} spec")
    return np.random.default_rng(spec.seed).random(spec.dims)


def _exact_distinct(rng, total: int, nnz: int) -> np.ndarray:
    """Sorted distinct linear indices, topped up to exactly nnz (synth.py:124-131 protocol)."""
    if nnz == total:
        return np.arange(total, dtype=np.int64)
    have = np.empty(0, dtype=np.int64)
    while have.size < nnz:
        fresh = rng.integers(0, total, size=nnz - have.size, dtype=np.int64)
        have = np.unique(np.concatenate([have, fresh]))
    return have


def _nonzero_uniform(rng, n: int) -> np.ndarray:
    vals = rng.random(n)
    while True:
        zero = vals == 0.0
        if not zero.any():
            return vals
        vals[zero] = rng.random(int(zero.sum()))


def gen_sparse3(spec: GenSpec) -> SparseCooTensor:
    """Order-3 tensor with exactly round(density * n1 n2 n3) distinct coordinates."""
    if spec.kind != "sparse3":
        raise GenerationError(f"gen_sparse3 got a {spec.kind!r} spec")
    nnz = spec.nnz
    if nnz == 0:
        raise GenerationError("degenerate spec: zero nonzeros requested")
    total = int(np.prod(spec.dims, dtype=object))
    rng = np.random.default_rng(spec.seed)
    lin = _exact_distinct(rng, total, nnz)      # indices first ...
    vals = _nonzero_uniform(rng, nnz)           # ... then values (pinned order)
    subs = np.column_stack(np.unravel_index(lin, spec.dims)).astype(np.int64, copy=False)
    return SparseCooTensor._from_canonical(subs, vals, spec.dims)


def derive_trial_seed(master: int, size_index: int, schedule_index: int) -> int:
    ss = np.random.SeedSequence((master, size_index, schedule_index))
    return int(ss.generate_state(1, np.uint64)[0])


def derive_arg_seed(trial_seed: int, arg_index: int) -> int:
    ss = np.random.SeedSequence((trial_seed, arg_index))
    return int(ss.generate_state(1, np.uint64)[0])


# BASELINE.json configs (1-based numbering as in BASELINE.md / SURVEY.md §8d)
CONFIGS = {
    1: {"name": "dot", "n": 10**6},
    2: {"name": "matvec", "rows": 4096, "cols": 4096},
    3: {"name": "ttv", "shape": (1000, 1000, 1000), "nnz": 10**6, "k": 2, "density": 0.001},
    4: {"name": "ttv_multi_dense", "shape": (20000,) * 4, "nnz": 10**8, "keep": 0},
    5: {"name": "ttv_zipf", "shape": (10**6, 10**5, 10**4), "nnz": 4 * 10**8, "k": 2, "zipf_s": 1.2},
}


def host_operands(config: int, master: int = DEFAULT_SEED, schedule_index: int = 0) -> dict:
    """Operands for configs 1-3, byte-identical to the reference's bench.build_operands
    (bench.py:366-384) for size index 0 and the given schedule index."""
    ts = derive_trial_seed(master, 0, schedule_index)
    if config == 1:
        n = CONFIGS[1]["n"]
        return {"x": gen_vector(GenSpec(derive_arg_seed(ts, 0), "vector", (n,))),
                "y": gen_vector(GenSpec(derive_arg_seed(ts, 1), "vector", (n,)))}
    if config == 2:
        r, c = CONFIGS[2]["rows"], CONFIGS[2]["cols"]
        return {"a": gen_matrix(GenSpec(derive_arg_seed(ts, 0), "matrix", (r, c))),
                "x": gen_vector(GenSpec(derive_arg_seed(ts, 1), "vector", (c,)))}
    if config == 3:
        cfg = CONFIGS[3]
        t = gen_sparse3(GenSpec(derive_arg_seed(ts, 0), "sparse3", cfg["shape"], cfg["density"]))
        x = gen_vector(GenSpec(derive_arg_seed(ts, 1), "vector", (cfg["shape"][cfg["k"]],)))
        return {"tensor": t, "x": x, "k0": cfg["k"]}
    raise GenerationError(f"config {config} is generated on the device (device.DeviceCoo.generate)")
