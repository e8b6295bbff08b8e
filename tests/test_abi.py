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


def test_peer_kernels_leave_room_for_a_second_peer_kernel():
    """Forward-progress rule of csrc/peer.cu: every peer kernel variant fits
    two blocks of 256 threads per SM (<= 128 registers, no spills) and does
    not release its stream's next kernel before its final barrier."""
    import subprocess
    from paper_2401_11202_b200.build import CSRC, FLAGS, INCLUDE, NVCC
    src = os.path.join(CSRC, "peer.cu")
    out = subprocess.run([NVCC, *FLAGS, "-c", src, "-o", os.devnull, "-Xptxas", "-v"],
                         capture_output=True, text=True, check=True)
    log = out.stdout + out.stderr
    regs = [int(r) for r in re.findall(r"Used (\d+) registers", log)]
    assert len(regs) >= 8
    assert max(regs) <= 128, regs
    assert not re.search(r"[1-9]\d* bytes spill stores", log)
    with open(src) as fh:
        code = fh.read()
    assert "SPX_PDL_ENTRY" not in code.split("namespace {", 1)[1]
    # the data-moving kernels fit two blocks per SM; the one-block barrier kernel is 32 threads
    assert code.count("__global__ void __launch_bounds__(256, 2)") == 3
    assert code.count("__global__ void __launch_bounds__(32) peer_barrier_kernel") == 1
    assert code.count("__global__") == 4
