"""Kernel backend selection -- the reference's plugin boundary (pkg/src/tenkern/backend.py:12-49).

The reference chooses between its compiled extension and an interpreted fallback.  This
package has exactly one backend, ``"b200"`` (the sm_100a kernels behind libtk_b200.so), and
deliberately no CPU fallback: if the library is missing the import fails loudly.
"""

from . import _kernels as _b200
from .errors import ConfigError

B200 = "b200"


def compiled_available() -> bool:
    """True when libtk_b200.so loads (it always must; there is no fallback)."""
    from . import _lib
    try:
        _lib.load()
    except ImportError:
        return False
    return True


def active_backend() -> str:
    return B200


def kernels(backend: str | None = None):
    """Return the kernel module for ``backend`` (default and only choice: "b200").

    Unknown names raise ConfigError, like the reference (backend.py:41-49).
    """
    if backend is None or backend == B200:
        return _b200
    raise ConfigError(f"unknown kernel backend {backend!r}")
