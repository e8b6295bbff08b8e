"""Arithmetic type at the drop-in boundary.

The reference computes in `np.result_type` of the inputs (spmd_interp.py:173,
interp.py:127) and constants adopt it (interp.py:39-41); the IR's element
kinds are f32 and i32 (ir.py:14).  The backend computes f32 and i32 (wrapping
int32 ufuncs, like numpy) and refuses every other result type instead of
computing it in another precision: f64 inputs, f32 mixed with i32 (numpy
promotes that to f64), int32 reduce-sum (np.sum widens to int64) and int32
exp (np.exp widens to f64)."""
import numpy as np
import pytest

from conftest import golden_cases, requires_gpu
from oracle import spmd_oracle as O

RULES = [c for c in golden_cases() if c["group"] == "rule" and c.get("error") is None and "exp" not in c["local_ir"]]

INT_PROGRAM = """func @main(%a: tensor<64x48xi32>, %b: tensor<48x80xi32>, %c: tensor<80xi32>, %d: tensor<64x80xi32>) -> (tensor<64x80xi32>, tensor<80xi32>, tensor<80x64xi32>) {
  %m = matmul %a, %b : tensor<64x80xi32>
  %cb = broadcast %c {dims = [1]} : tensor<64x80xi32>
  %s = add %m, %cb : tensor<64x80xi32>
  %k = constant 3.7 : tensor<64x80xi32>
  %t = mul %s, %k : tensor<64x80xi32>
  %n = neg %d : tensor<64x80xi32>
  %u = add %t, %n : tensor<64x80xi32>
  %sq = mul %u, %u : tensor<64x80xi32>
  %mx = reduce %sq {dims = [0], monoid = max} : tensor<80xi32>
  %tr = transpose %u {perm = [1, 0]} : tensor<80x64xi32>
  return %u, %mx, %tr
}
"""


def _pkg():
    import paper_2401_11202_b200 as pkg
    return pkg


def test_f64_and_mixed_inputs_raise_typeerror():
    pkg = _pkg()
    case = next(c for c in golden_cases() if c["key"] == "rule_rs_raw")
    m = pkg.parse_module(case["local_ir"])
    spec = pkg.ShardingSpec.from_json(case["sharding"])
    f = m.func("main")
    ins64 = {n: np.zeros(t.dims, np.float64) for n, t in f.args}
    with pytest.raises(TypeError, match="float64"):
        pkg.spmd_interpret(m, spec, ins64)
    d = pkg.parse_module(INT_PROGRAM)
    fd = d.func("main")
    mixed = {n: np.zeros(t.dims, np.int32 if i else np.float32) for i, (n, t) in enumerate(fd.args)}
    with pytest.raises(TypeError, match="float64"):
        pkg.interpret(d, mixed)


@pytest.mark.parametrize("body,what", [
    ("%r = reduce %x {dims = [0]} : tensor<8xi32>", "int64"),
    ("%r = exp %x : tensor<4x8xi32>", "float64"),
])
def test_int32_widening_ops_refused(body, what):
    from paper_2401_11202_b200.executable import Executable
    pkg = _pkg()
    rt = "tensor<8xi32>" if "reduce" in body else "tensor<4x8xi32>"
    text = f"func @main(%x: tensor<4x8xi32>) -> {rt} {{\n  {body}\n  return %r\n}}\n"
    with pytest.raises(TypeError, match=what):
        Executable(pkg.parse_module(text), devices=[0], dry=True, dtype=np.int32)


def test_int32_constant_cast_like_numpy():
    """constant 3.7 in an int32 call is np.full(..., 3.7, int32) = 3."""
    from paper_2401_11202_b200.plan import Compiler
    pkg = _pkg()
    c = Compiler(pkg.parse_module(INT_PROGRAM), dtype=np.int32).compile()
    assert c.desc["k"].value == np.full((1,), 3.7, np.int32)[0] == 3


@pytest.mark.gpu
@requires_gpu
@pytest.mark.parametrize("case", RULES, ids=lambda c: c["key"])
def test_int32_collectives_bitexact(case):
    """Every collective rule program with int32 inputs (all_slice, all_gather,
    all_reduce, reduce_scatter, all_to_all, multi-axis layouts, the max monoid):
    bit-exact against the oracle, dtype int32."""
    pkg = _pkg()
    m = pkg.parse_module(case["local_ir"])
    spec = pkg.ShardingSpec.from_json(case["sharding"])
    base = pkg.parse_module(case["dense_ir"]) if "dense_ir" in case else m
    rng = np.random.default_rng(7)
    ins = {n: rng.integers(-2**31, 2**31 - 1, t.dims, dtype=np.int64).astype(np.int32)
           for n, t in base.func("main").args}
    want = O.spmd_interpret(m, spec, ins)
    got = pkg.spmd_interpret(m, spec, ins)
    for g, w in zip(got, want):
        assert g.dtype == w.dtype == np.int32
        np.testing.assert_array_equal(g, w)


@pytest.mark.gpu
@requires_gpu
def test_int32_arithmetic_bitexact():
    """matmul (wrapping int32 accumulation), broadcast add, constant cast,
    mul/neg wraparound, reduce max, transpose: bit-exact with numpy."""
    pkg = _pkg()
    m = pkg.parse_module(INT_PROGRAM)
    rng = np.random.default_rng(3)
    ins = {n: rng.integers(-2**31, 2**31 - 1, t.dims, dtype=np.int64).astype(np.int32)
           for n, t in m.func("main").args}
    with np.errstate(all="ignore"):
        want = O.interpret(m, ins)
    got = pkg.interpret(m, ins)
    for g, w in zip(got, want):
        assert g.dtype == w.dtype == np.int32
        np.testing.assert_array_equal(g, w)
