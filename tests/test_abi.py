"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/ldpc.h declares (no GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ldpc.h")).read()
    return sorted(set(re.findall(r"LDPC_API\s+[\w\s\*]*?\b(ldpc_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2507_10424_b200 import build

    return build.build()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("ldpc_prepare_dense", "ldpc_prepare_coo", "ldpc_decode", "ldpc_decode_host", "ldpc_info",
                 "ldpc_destroy", "ldpc_status_string"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ldpc_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_binding_matches_header(lib_path):
    from paper_2507_10424_b200 import _lib

    lib = _lib.load()
    assert lib.ldpc_abi_version() == 1
    assert set(_lib.SIGNATURES) == set(declared_symbols())
    assert lib.ldpc_status_string(-3).decode() == "H has a row of degree < 2"
    # argument errors return before touching the device
    h = ctypes.c_void_p()
    assert lib.ldpc_prepare_dense(None, 5, 10, 0, None, ctypes.byref(h)) == -1
    assert lib.ldpc_decode(None, None, 10, 5, None, None, None, None, None, None) == -1


def test_kernels_are_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_touch_the_oracle():
    """The product package never imports or links the oracle (parity would be void otherwise)."""
    pkg = os.path.join(ROOT, "paper_2507_10424_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.lower(), f
