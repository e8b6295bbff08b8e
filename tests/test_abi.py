"""The C-ABI library builds, loads and exports every symbol include/spindle_b200.h
declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

from conftest import ROOT


def test_header_symbols_exported():
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.build import build
    build()
    lib = ctypes.CDLL(R.LIB_PATH)
    with open(os.path.join(ROOT, "include", "spindle_b200.h")) as fh:
        hdr = fh.read()
    declared = set(re.findall(r"^\s*(?:const\s+char\*|int)\s+(spx_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert declared >= set(R.EXPORTS)


def test_record_abi_sizes_match():
    from paper_2401_11202_b200 import runtime as R
    lib = R.load()
    R.check_abi(lib)
    assert lib.spx_version() == 1
