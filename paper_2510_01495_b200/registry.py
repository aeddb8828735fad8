"""Registration of the B200 kernel module in the reference's benchmark registry.

The reference's harness looks implementations up by label (``ImplEntry`` +
``register_implementation``, /root/reference/pkg/src/tenkern/bench.py:191-215); its built-in
``native-loop`` label wraps the compiled module's self-timed entry points
(``_native_thunk``, bench.py:248-257) and the companion package registers host-side labels
the same way (/root/reference/pkg/hostbench/src/tenhost/registry.py:85-115).  ``register()``
adds, next to them:

* ``b200`` -- self-timed like ``native-loop``: the thunks call this package's
  ``dot_timed`` / ``matvec_timed`` / ``ttv_timed`` (the native clock of libtk_b200.so around
  the host-buffer C-ABI call, H2D and D2H included);
* ``b200-via-ffi`` (when ``tenhost`` is importable) -- host-timed like ``native-via-ffi``:
  ``tenhost.BoundKernelSet(kernel_module=kernels())`` (bindings.py:40-79) crossing the boundary,
  plus ``host_reassemble_sparse`` for TTV, exactly the reference label's timed region.

The reference package is imported only inside ``register()``: this package does not depend on
it.  A child interpreter (the reference's first-call overhead estimator spawns ``python -m
tenhost._child``) must call ``register()`` before the harness runs -- see INTEGRATION.md.
"""

from __future__ import annotations

LABEL = "b200"
LABEL_FFI = "b200-via-ffi"


def available() -> bool:
    """The library loads and a CUDA device is visible."""
    from . import _lib
    try:
        return _lib.device_count() > 0
    except (ImportError, OSError):
        return False


def _unavailable_reason() -> str:
    from . import _lib
    try:
        _lib.load()
    except ImportError as exc:
        return str(exc)
    return "no CUDA device visible (libtk_b200.so has no CPU fallback)"


def _b200_thunk(experiment, data, checked):
    """Mirror of the reference's _native_thunk (bench.py:248-257) for the B200 module."""
    from .backend import kernels
    K = kernels()
    if experiment == "dot":
        x, y = data["x"], data["y"]
        return lambda: K.dot_timed(x, y, checked=checked)
    if experiment.startswith("matvec"):
        a, x = data["a"], data["x"]
        return lambda: K.matvec_timed(a, x, checked=checked)
    t, xv, k0 = data["tensor"], data["x"], data["k0"]
    return lambda: K.ttv_timed(t.subs, t.vals, t.shape, xv, k0)


def _ffi_thunk(experiment, data, checked):
    """Mirror of tenhost's _ffi_thunk (tenhost/registry.py:41-60), unchecked form, over the
    B200 module bound through the reference's own BoundKernelSet."""
    from tenhost.bindings import BoundKernelSet
    from tenhost.hosttensor import host_reassemble_sparse
    from .backend import kernels
    bks = BoundKernelSet(kernel_module=kernels())
    if experiment == "dot":
        x, y = data["x"], data["y"]
        return lambda: bks.dot(x, y)
    if experiment.startswith("matvec"):
        a, x = data["a"], data["x"]
        return lambda: bks.matvec(a, x)
    t, xv, k0 = data["tensor"], data["x"], data["k0"]
    return lambda: host_reassemble_sparse(bks.ttv(t.subs, t.vals, t.shape, xv, k0), validate=False)


def register() -> list:
    """Install the B200 labels in the reference's registry (idempotent); returns the labels."""
    import tenkern
    from tenkern import ImplEntry, register_implementation
    reason = _unavailable_reason() if not available() else ""
    register_implementation(ImplEntry(label=LABEL, self_timed=True, available=available,
                                      unavailable_reason=reason, make_thunk=_b200_thunk))
    labels = [LABEL]
    try:
        import tenhost  # noqa: F401  (its import registers the reference's host-side labels)
    except ImportError:
        return labels
    register_implementation(ImplEntry(label=LABEL_FFI, self_timed=False, available=available,
                                      unavailable_reason=reason, make_thunk=_ffi_thunk,
                                      experiments=tenkern.EXPERIMENTS))
    labels.append(LABEL_FFI)
    return labels


def estimate_overhead(size: int, *, label: str = LABEL, **kwargs):
    """The reference's own first-call overhead estimator (tenhost.overhead.estimate_overhead,
    overhead.py:76-175) run for a B200 label.  Its children are started through the
    ``_child`` shim (a one-line interpreter wrapper that registers the labels before running
    ``tenhost._child``); everything else -- the schedule, the fresh processes, the discard
    rules, the arithmetic -- is the reference's."""
    import os
    import stat
    import sys
    import tempfile
    from tenhost import overhead
    register()
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory(prefix="tk-b200-child-") as tmp:
        exe = os.path.join(tmp, "python-b200")
        with open(exe, "w") as fh:
            fh.write(f"#!/bin/sh\nexec {sys.executable} -m paper_2510_01495_b200._child \"$@\"\n")
        os.chmod(exe, os.stat(exe).st_mode | stat.S_IEXEC)
        paths = [repo] + [p for p in sys.path if p and os.path.isdir(os.path.join(p, "tenhost"))]
        old_exe, old_pp = sys.executable, os.environ.get("PYTHONPATH")
        os.environ["PYTHONPATH"] = os.pathsep.join(paths + ([old_pp] if old_pp else []))
        sys.executable = exe
        try:
            return overhead.estimate_overhead(label, size, **kwargs)
        finally:
            sys.executable = old_exe
            if old_pp is None:
                os.environ.pop("PYTHONPATH", None)
            else:
                os.environ["PYTHONPATH"] = old_pp
