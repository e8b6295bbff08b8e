"""Run-time specialised elementwise kernels (csrc/ew_jit.cu), CPU side: the
generator emits a kernel for every f32 record shape the plan compiler produces
and NVRTC compiles each one for sm_100a (no GPU needed).  The GPU parity of
the compiled kernels is in test_gpu_parity.py::test_ew_jit_bitexact."""
import ctypes as C
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2401_11202_b200 import runtime as R  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    lib = R.load()
    if not lib.spx_ew_jit_available():
        pytest.skip("NVRTC not loadable here")
    return lib


def _source(lib, p) -> str:
    buf = C.create_string_buffer(1 << 20)
    n = lib.spx_ew_jit_source(C.byref(p), buf, len(buf))
    assert n > 0, lib.spx_last_error()
    return buf.value.decode()


def _compile(lib, p):
    rc = lib.spx_ew_jit_compile(C.byref(p))
    assert rc == 0, lib.spx_last_error()


def _params(dims, strides, prog, n_out=1, out_regs=(0,), imm=None, vec=None):
    p = R.EwParams()
    p.base, p.dev_stride, p.ndev = 1 << 20, 1 << 30, 1
    p.rank = len(dims)
    for i, d in enumerate(dims):
        p.dims[i] = d
    p.numel = int(np.prod(dims)) if dims else 1
    p.n_in = len(strides)
    for j, st in enumerate(strides):
        p.inp[j].off = 4096 * j
        for i, s in enumerate(st):
            p.inp[j].stride[i] = s
    p.n_out = n_out
    for o in range(n_out):
        p.out_off[o] = 1 << 24 + o
        p.out_reg[o] = out_regs[o]
    p.n_prog = len(prog)
    for i, (op, a, b, d) in enumerate(prog):
        p.prog[i].op, p.prog[i].a, p.prog[i].b, p.prog[i].dst = op, a, b, d
        p.imm[i] = (imm or [0.5] * len(prog))[i]
    if vec is None:
        vec = bool(dims) and dims[-1] % 4 == 0 and all(st[-1] in (0, 1) for st in strides)
    p.vec = int(vec)
    p.dtype = R.DT_F32 if hasattr(R, "DT_F32") else 0
    return p


OP = R.OP


def test_every_opcode_compiles(lib):
    prog = [(OP["ADD"], 0, 1, 2), (OP["MUL"], 2, 0, 3), (OP["NEG"], 3, 0, 3), (OP["EXP"], 3, 0, 4),
            (OP["MAX"], 4, 1, 5), (OP["IMM"], 0, 0, 6), (OP["ADDI"], 5, 0, 5), (OP["MULI"], 5, 0, 5),
            (OP["IADD"], 5, 0, 7), (OP["IMUL"], 7, 0, 7), (OP["MOV"], 7, 0, 8), (OP["ADD"], 8, 6, 0)]
    p = _params([256, 128], [[128, 1], [0, 1]], prog, n_out=2, out_regs=(0, 5))
    src = _source(lib, p)
    # IEEE ops stay separate roundings (no FMA contraction): the bit-exact contract
    for tok in ("__fadd_rn", "__fmul_rn", "expf(", "fmx("):
        assert tok in src
    _compile(lib, p)


@pytest.mark.parametrize("dims,strides", [
    ([], [[]]),                                           # rank 0 (a scalar)
    ([1000], [[1], [0]]),                                 # ragged, scalar broadcast
    ([2048, 2, 16, 2, 512], [[8192, 0, 512, 0, 1]]),      # nearest upsample (C4)
    ([64, 48, 32], [[1, 64 * 32, 64]]),                   # a transpose: no float4 path
    ([3, 5, 7, 9, 11, 13], [[15015, 3003, 429, 143, 13, 1], [0, 0, 0, 0, 0, 0]]),
    ([33, 17], [[17, 1], [1, 0], [0, 1]]),                # odd sizes, row + column broadcasts
])
def test_geometries_compile(lib, dims, strides):
    prog = [(OP["MUL"], 0, 0, 0)] if len(strides) == 1 else [(OP["ADD"], 0, 1, 0)] + \
        [(OP["MUL"], 0, j, 0) for j in range(2, len(strides))]
    p = _params(dims, strides, prog)
    src = _source(lib, p)
    if dims:
        # the broadcast (stride-0) dimensions never enter the address arithmetic
        for j, st in enumerate(strides):
            line = next(l for l in src.splitlines() if l.strip().startswith(f"const i64 o{j} ="))
            for k, s in enumerate(st[:-1]):
                assert (f"i{k} *" in line) == (s != 0), (line, st)
    _compile(lib, p)


def test_wide_records_use_64bit_indices(lib):
    p = _params([1 << 16, 1 << 16], [[1 << 16, 1]], [(OP["NEG"], 0, 0, 0)])
    assert p.numel >= 1 << 31
    src = _source(lib, p)
    assert "const u64 n =" in src
    _compile(lib, p)


def test_eight_inputs_four_outputs(lib):
    prog = [(OP["ADD"], j, j + 1, j + 1) for j in range(7)]
    p = _params([4096], [[1]] * 8, prog, n_out=4, out_regs=(7, 6, 5, 0))
    _compile(lib, p)


def test_cache_by_source(lib):
    a, b = C.c_int(), C.c_int()
    p = _params([512, 64], [[64, 1], [0, 1]], [(OP["ADD"], 0, 1, 0), (OP["MULI"], 0, 0, 0)])
    _compile(lib, p)
    lib.spx_ew_jit_stats(C.byref(a), C.byref(b))
    n0 = a.value
    p.inp[0].off += 64           # offsets and immediates are parameters: same kernel
    p.imm[1] = 3.0
    _compile(lib, p)
    lib.spx_ew_jit_stats(C.byref(a), C.byref(b))
    assert a.value == n0
    p.dims[0] = 1024             # the shape is compiled in: a new kernel
    p.numel = 1024 * 64
    _compile(lib, p)
    lib.spx_ew_jit_stats(C.byref(a), C.byref(b))
    assert a.value == n0 + 1


def test_bad_records_rejected(lib):
    p = _params([64], [[1]], [(OP["ADD"], 0, 13, 0)])
    assert lib.spx_ew_jit_compile(C.byref(p)) != 0
    assert b"slot" in lib.spx_last_error()
    p = _params([64], [[1]], [(99, 0, 0, 0)])
    assert lib.spx_ew_jit_compile(C.byref(p)) != 0


def test_config_programs_generic_records_compile(lib):
    """Every elementwise record of the U-Net analog outside the static catalog
    (its upsample broadcasts and gradient products) compiles."""
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.programs import load_program
    prog = load_program("c4_unet_dense")
    ex = Executable(prog.dense, devices=[0], dry=True)
    match = getattr(lib, "_Z19spx_ew_static_matchRK13spx_ew_params")
    match.restype = C.c_int
    n = 0
    for kind, p in ex.records():
        if kind == R.K_EW and not (p.rank <= 2 and match(C.byref(p)) >= 0):
            _compile(lib, p)
            n += 1
    assert n >= 4


def test_fused_split_variant_compiles(lib):
    """The elementwise records of the U-Net analog whose output is split for a
    3xFP16 GEMM right after them (rank > 2: outside the static kernels) get
    the fused-split variant (4-CTA clusters, pieces bit-identical to the
    standalone split), with and without the fp32 store."""
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.programs import load_program
    prog = load_program("c4_unet_dense")
    ex = Executable(prog.dense, devices=[0], dry=True)
    recs = ex.records()
    match = getattr(lib, "_Z19spx_ew_static_matchRK13spx_ew_params")
    match.restype = C.c_int
    n = 0
    for (ka, a), (kb, b) in zip(recs, recs[1:]):
        if ka != R.K_EW or kb != R.K_SPLIT or (a.rank <= 2 and match(C.byref(a)) >= 0):
            continue
        which = [a.out_off[j] for j in range(a.n_out)].index(b.src_off) if b.src_off in \
            [a.out_off[j] for j in range(a.n_out)] else -1
        if which < 0:
            continue
        buf = C.create_string_buffer(1 << 20)
        for skip in (0, 1):
            assert lib.spx_ew_jit_split_source(C.byref(a), which, skip, buf, len(buf)) > 0
            src = buf.value.decode()
            assert "__cluster_dims__(4, 1, 1)" in src and "cvt.rn.f16x2.f32" in src
            rc = lib.spx_ew_jit_split_compile(C.byref(a), C.byref(b), which, skip)
            assert rc == 0, lib.spx_last_error()
        n += 1
    assert n >= 2
