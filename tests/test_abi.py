"""The C-ABI library builds for sm_100a, loads, and exports every entry point
declared in include/dlmpc.h (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re
import subprocess

import pytest

import build
from paper_2103_14990_b200 import device

HEADER = os.path.join(os.path.dirname(build.__file__), "include", "dlmpc.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\*\s]+?\b(dlmpc_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    return build.build()


def test_header_declares_the_abi():
    names = declared_functions()
    assert set(device.EXPORTS) == set(names), set(device.EXPORTS) ^ set(names)


def test_library_loads_and_exports_all_symbols(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_code(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_fp64_tensor_cores(lib_path):
    """The fast Ψ path issues DMMA (FP64 mma.sync); tcgen05 has no f64 kind."""
    out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "DMMA" in out


def test_no_device_error_is_loud(lib_path):
    """Without a GPU the create call fails with a clear status, never silently."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    lib = device.load_library()
    h = ctypes.c_void_p()
    rc = lib.dlmpc_create(ctypes.byref(device._Problem()), 0, ctypes.byref(h))
    assert rc != 0
    assert lib.dlmpc_global_error()
