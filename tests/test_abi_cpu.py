"""The C-ABI library loads here (no GPU) and exports every symbol include/tk_b200.h declares."""

import os
import re
import subprocess

import pytest

from conftest import REPO
from paper_2510_01495_b200 import _lib, errors

HEADER = os.path.join(REPO, "include", "tk_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_expected_surface():
    syms = declared_symbols()
    for s in ("tk_ttv_f64_device", "tk_ttv_f64_host", "tk_dot_f64_host", "tk_matvec_f64_host",
              "tk_ttv_dense_f64_device", "tk_group_sum_f64_host", "tk_last_error", "tk_ttv_workspace",
              "tk_ttv_f64_device_timed", "tk_dot_f64_device_timed", "tk_matvec_f64_device_timed",
              "tk_multi_init", "tk_multi_ttv_f64", "tk_multi_free", "tk_ttv_dense_f64_device_peers"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (tk_\w+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert hasattr(lib, s)
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_bulk_copy_engine():
    # the streaming TTV kernels stage tiles with cp.async.bulk (TMA engine): SASS UBLKCP
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in out


def test_version_and_error_string():
    lib = _lib.load()
    assert lib.tk_version() >= 100
    assert isinstance(lib.tk_last_error(), bytes)


@pytest.mark.skipif(_lib.device_count() > 0, reason="GPU present: covered by -m gpu tests")
def test_compute_fails_loudly_without_a_gpu():
    import numpy as np
    from paper_2510_01495_b200 import _kernels as kernels
    with pytest.raises(errors.DeviceError):
        kernels.dot(np.ones(4), np.ones(4))
    with pytest.raises(errors.DeviceError):
        kernels.ttv_raw(np.zeros((1, 3), dtype=np.int64), np.ones(1), (2, 2, 2), np.ones(2), 2)


def test_structural_guards_raise_before_any_device_work():
    import numpy as np
    from paper_2510_01495_b200 import _kernels as kernels
    subs = np.zeros((1, 3), dtype=np.int64)
    with pytest.raises(errors.ModeError):
        kernels.ttv_raw(subs, [1.0], (8, 8, 8), np.ones(8), 3)
    with pytest.raises(errors.DimensionError):
        kernels.ttv_raw(subs, [1.0], (8, 8, 8), np.ones(5), 1)
    with pytest.raises(errors.OrderError):
        kernels.ttv_raw(np.zeros((1, 1), dtype=np.int64), [1.0], (4,), np.ones(4), 0)
    with pytest.raises(errors.DimensionError):
        kernels.dot(np.ones(3), np.ones(4))
    with pytest.raises(errors.DimensionError):
        kernels.matvec(np.ones((2, 3)), np.ones(2))


def test_ttv_workspace_is_host_arithmetic():
    """tk_ttv_workspace needs no GPU: an upper bound that grows with nnz and rejects bad sizes."""
    import ctypes
    lib = _lib.load()
    b1, b2 = ctypes.c_size_t(0), ctypes.c_size_t(0)
    assert lib.tk_ttv_workspace(3, 1_000_000, 2, ctypes.byref(b1)) == 0
    assert lib.tk_ttv_workspace(3, 4 * 10**8, 2, ctypes.byref(b2)) == 0
    assert b2.value > b1.value >= 1_000_000 * 8 * 3
    assert lib.tk_ttv_workspace(1, 10, 0, ctypes.byref(b1)) != 0
