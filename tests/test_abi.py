"""The C-ABI libraries load and export every symbol include/e2sched.h
declares (no compute calls: CPU-safe)."""
from __future__ import annotations

import ctypes
import os
import re

from paper_2407_00023_b200 import abi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "e2sched.h")).read()
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(e2_[a-z_0-9]+)\(", src, re.M))


def test_header_and_binding_agree():
    assert header_symbols() == set(abi.DECLARED_SYMBOLS)


def test_product_library_exports_abi():
    assert os.path.exists(abi.PRODUCT_SO), "run __graft_entry__.build()"
    lib = ctypes.CDLL(abi.PRODUCT_SO)
    for name in header_symbols():
        assert hasattr(lib, name), name
    lib.e2_backend.restype = ctypes.c_char_p
    assert lib.e2_backend() == b"b200"


def test_checker_libraries_export_abi(hostsim_lib, ref_lib):
    for name in header_symbols():
        assert hasattr(hostsim_lib, name), name
    for name in header_symbols() - set(abi.PRODUCT_ONLY):
        assert hasattr(ref_lib, name), name


def test_product_has_no_host_fallback():
    """The shipped .so contains sm_100a code and reports the b200 backend."""
    data = open(abi.PRODUCT_SO, "rb").read()
    assert b"sm_100a" in data or b"compute_100a" in data
    assert b"hostsim" not in data
