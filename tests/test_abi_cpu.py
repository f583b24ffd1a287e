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


def test_library_links_completely():
    # every symbol of the library's own namespace is defined inside it (a declaration left without
    # a definition loads lazily here and fails only at the first call on the GPU box)
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    L = ctypes.CDLL(_native.LIB_PATH, mode=os.RTLD_NOW)
    assert L is not None
    out = subprocess.run(["nm", "-D", "--undefined-only", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "fpfp" not in out, [ln for ln in out.splitlines() if "fpfp" in ln]


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


def test_missing_library_fails_loudly(tmp_path):
    # the binding has no fallback: a missing libfastpfp.so is an error at first use
    code = ("import paper_1207_1114_b200 as F\n"
            "try:\n    F.lib()\nexcept Exception as e:\n    print('RAISED', type(e).__name__)\n"
            "else:\n    print('LOADED')\n")
    env = dict(os.environ, FASTPFP_LIB=str(tmp_path / "absent.so"))
    out = subprocess.run([os.sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__)))).stdout
    assert "RAISED" in out, out


def test_no_device_is_an_error_not_a_cpu_fallback():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    st = _native.lib().fastpfp_create(8, 8, 0, ctypes.byref(h))
    assert st in (_native.ENODEV, _native.ECUDA), st


def test_product_package_never_imports_the_oracle():
    # the oracle is test infrastructure: nothing under paper_1207_1114_b200/ may import it
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1207_1114_b200")
    offenders = []
    for dp, _, files in os.walk(root):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dp, f)).read()
                if "import oracle" in src or "from oracle" in src:
                    offenders.append(os.path.join(dp, f))
    assert not offenders, offenders
    # and the CUDA sources share no header with it
    csrc = os.path.join(root, "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        assert "oracle" not in "".join(l for l in src.splitlines() if l.startswith("#include")), f
