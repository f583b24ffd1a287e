"""CPU-side checks of the C-ABI library: it builds, loads without a GPU and exports every symbol
that include/fastpfp.h declares; host-side argument validation that needs no device."""
import ctypes
import os
import subprocess

import pytest

from paper_1207_1114_b200 import _native


def test_header_declares_the_north_star_calls():
    names = _native.declared_symbols()
    for call in ("fastpfp_create", "fastpfp_set_graphs", "fastpfp_iterate", "fastpfp_discretize",
                 "fastpfp_destroy"):
        assert call in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    L = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in _native.declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    for s in _native.declared_symbols():
        assert f" T {s}" in out, s


def test_library_is_sm100a_code():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_static_calls_without_device():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    L = _native.lib()
    assert L.fastpfp_abi_version() == 1
    assert L.fastpfp_status_string(_native.ESYM).decode().startswith("adjacency")
    h = ctypes.c_void_p()
    # argument validation happens before any device call
    assert L.fastpfp_create(0, 5, 0, ctypes.byref(h)) == _native.EINVAL
    assert L.fastpfp_create(5, 5, -1, ctypes.byref(h)) == _native.EINVAL
