"""tk-b200: B200-native (sm_100a) drop-in for the reference's tensor kernels (arXiv 2510.01495).

Mirrors the public surface of the reference package ``tenkern`` that sits on the hot path
(pkg/src/tenkern/__init__.py:54-109): dense ``dot`` / ``matvec``, the canonical
``SparseCooTensor``, ``ttv`` with its ``TtvRawResult`` triple, the helpers, the error
classes, seeded generators and the kernel-module protocol (``kernels()``).  All arithmetic
runs in libtk_b200.so (hand-written CUDA for sm_100a); there is no CPU fallback.
"""

from .backend import active_backend, compiled_available, kernels
from .dense import as_matrix, as_vector, dot, matvec
from .errors import (
    ConfigError,
    DeviceError,
    DimensionError,
    GenerationError,
    IntegrityError,
    ModeError,
    OrderError,
    SizeCapError,
    TenkernError,
)
from .sparse import (
    SparseCooTensor,
    TtvRawResult,
    densify,
    mttkrp,
    set_difference,
    ttv,
    unique_rows_accumulate,
)
from .synth import GENERATOR, GenSpec, gen_matrix, gen_sparse3, gen_vector

__version__ = "0.1.0"

__all__ = [
    "__version__",
    "active_backend",
    "compiled_available",
    "kernels",
    "TenkernError",
    "DimensionError",
    "ModeError",
    "OrderError",
    "SizeCapError",
    "GenerationError",
    "ConfigError",
    "IntegrityError",
    "DeviceError",
    "as_vector",
    "as_matrix",
    "dot",
    "matvec",
    "SparseCooTensor",
    "TtvRawResult",
    "ttv",
    "set_difference",
    "unique_rows_accumulate",
    "densify",
    "mttkrp",
    "GENERATOR",
    "GenSpec",
    "gen_vector",
    "gen_matrix",
    "gen_sparse3",
]
