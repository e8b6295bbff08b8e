"""GPU parity: the CUDA path against the reference's golden outputs and the
oracle restatement, through the drop-in `spmd_interpret` / `interpret`.

Bars: bit-exact for data movement and fp32 add/mul/neg;
<= 1e-5 max-normalised relative error (`relative_error`, spmd_interp.py:25-31)
for matmul, reduce, all_reduce/reduce_scatter sums and exp.  All outputs are
checked finite first.
"""
import numpy as np
import pytest

from conftest import TOL, case_expected, case_inputs, golden_cases, requires_gpu
from oracle import spmd_oracle as O

pytestmark = [pytest.mark.gpu, requires_gpu]

CASES = golden_cases()


def _pkg():
    import paper_2401_11202_b200 as pkg
    return pkg


@pytest.mark.parametrize("case", [c for c in CASES if "local_ir" in c], ids=lambda c: c["key"])
def test_spmd_golden(case):
    pkg = _pkg()
    m = pkg.parse_module(case["local_ir"])
    spec = pkg.ShardingSpec.from_json(case["sharding"])
    base = pkg.parse_module(case["dense_ir"]) if "dense_ir" in case else m
    for s in case["seeds"]:
        ins = case_inputs(case, base, s)
        if case.get("error") == "DivergenceError":
            with pytest.raises(pkg.DivergenceError):
                pkg.spmd_interpret(m, spec, ins)
            continue
        got = pkg.spmd_interpret(m, spec, ins)
        for g, w in zip(got, case_expected(case, s, "spmd")):
            assert np.all(np.isfinite(g))
            if case["group"] == "rule" and "exp" not in case["local_ir"]:
                np.testing.assert_array_equal(g, w)
            else:
                assert O.relative_error(g, w) < TOL


@pytest.mark.parametrize("case", [c for c in CASES if "dense_ir" in c], ids=lambda c: c["key"])
def test_dense_golden(case):
    pkg = _pkg()
    m = pkg.parse_module(case["dense_ir"])
    for s in case["seeds"]:
        ins = case_inputs(case, m, s)
        got = pkg.interpret(m, ins)
        for g, w in zip(got, case_expected(case, s, "dense")):
            assert np.all(np.isfinite(g))
            if case["key"] in ("op_add", "op_mul", "op_neg", "op_tag", "op_transpose2", "op_transpose3",
                               "op_reshape1", "op_reshape2", "op_reshape3", "op_broadcast0",
                               "op_broadcast1", "op_broadcast2", "op_reduce1max", "op_reduce0max3"):
                np.testing.assert_array_equal(g, w)
            else:
                assert O.relative_error(g, w) < TOL


def _mm_module(M, K, N, at=False, bt=False):
    """matmul with optionally transposed operands (stored transposed, then a
    `transpose` op feeds the matmul -- the pattern of matmul_grads, models.py:64-71)."""
    a_t = f"tensor<{K}x{M}xf32>" if at else f"tensor<{M}x{K}xf32>"
    b_t = f"tensor<{N}x{K}xf32>" if bt else f"tensor<{K}x{N}xf32>"
    lines = [f"func @main(%a: {a_t}, %b: {b_t}) -> tensor<{M}x{N}xf32> {{"]
    a, b = "%a", "%b"
    if at:
        lines.append(f"  %at = transpose %a {{perm = [1, 0]}} : tensor<{M}x{K}xf32>")
        a = "%at"
    if bt:
        lines.append(f"  %bt = transpose %b {{perm = [1, 0]}} : tensor<{K}x{N}xf32>")
        b = "%bt"
    lines.append(f"  %c = matmul {a}, {b} : tensor<{M}x{N}xf32>")
    lines.append("  return %c\n}\n")
    return _pkg().parse_module("\n".join(lines))


GEMM_SHAPES = [
    (128, 128, 128), (256, 512, 384), (1024, 1024, 1024), (2048, 1024, 4096),
    (1024, 2048, 1024), (192, 96, 160), (130, 70, 200), (1024, 128, 1024),
    (128, 8192, 256), (256, 32768, 64),      # few tiles, long K: split-K partials + reduction
]


@pytest.mark.parametrize("at,bt", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("shape", GEMM_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_gemm_tcgen05_3xtf32(shape, at, bt):
    """tcgen05 3xTF32 GEMM vs float64 numpy: <= 1e-5 max-normalised (fp32 parity)."""
    pkg = _pkg()
    M, K, N = shape
    if shape == (130, 70, 200) and (at or bt):
        pytest.skip("TMA needs 16B row pitch; 130/70 rows exercise the SIMT fallback elsewhere")
    rng = np.random.default_rng(hash(shape) % 1000)
    a = rng.standard_normal((K, M) if at else (M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if bt else (K, N)).astype(np.float32)
    m = _mm_module(M, K, N, at, bt)
    A = a.T if at else a
    B = b.T if bt else b
    want = A.astype(np.float64) @ B.astype(np.float64)
    path = 0 if (M % 4 or K % 4 or N % 4) else 1
    (got,) = pkg.interpret(m, {"a": a, "b": b}, gemm_path=path)
    assert np.all(np.isfinite(got))
    err = O.relative_error(got, want)
    assert err < TOL, err
    # and vs numpy's own float32 matmul (the oracle's arithmetic)
    assert O.relative_error(got, A @ B) < TOL


@pytest.mark.parametrize("at,bt", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("shape", [s for s in GEMM_SHAPES if s != (130, 70, 200)] + [(256, 72, 136), (320, 200, 96)],
                         ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("bn", ["128", "256"])
def test_gemm_h3_block_scaled(shape, at, bt, bn, monkeypatch):
    """Block-scaled 3xFP16 GEMM (gemm_h3.cu) vs float64: <= 1e-5 max-normalised,
    both tile widths (BN = 128 / 256 output columns per CTA pair)."""
    monkeypatch.setenv("SPX_H3_BN", bn)
    pkg = _pkg()
    M, K, N = shape
    rng = np.random.default_rng(hash(shape) % 1000 + 7)
    a = rng.standard_normal((K, M) if at else (M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if bt else (K, N)).astype(np.float32)
    A = a.T if at else a
    B = b.T if bt else b
    (got,) = pkg.interpret(_mm_module(M, K, N, at, bt), {"a": a, "b": b}, gemm_path=3)
    assert np.all(np.isfinite(got))
    want = A.astype(np.float64) @ B.astype(np.float64)
    assert O.relative_error(got, want) < TOL
    assert O.relative_error(got, A @ B) < TOL


@pytest.mark.parametrize("at,bt", [(False, False), (True, False), (False, True)])
@pytest.mark.parametrize("shape", [(512, 4096, 1024), (256, 2048, 512), (128, 8192, 256), (1024, 1024, 1024)],
                         ids=lambda s: "x".join(map(str, s)))
def test_gemm_h3_splitk(shape, at, bt, monkeypatch):
    """Few-tile GEMMs split K across CTA pairs (opt-in; the last unit of each
    slice folds the partials in split order): within 1e-5, bit-identical
    across runs, and close to the unsplit kernel."""
    monkeypatch.setenv("SPX_H3_SPLITK", "8")
    pkg = _pkg()
    M, K, N = shape
    rng = np.random.default_rng(5)
    a = rng.standard_normal((K, M) if at else (M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if bt else (K, N)).astype(np.float32)
    A = a.T if at else a
    B = b.T if bt else b
    m = _mm_module(M, K, N, at, bt)
    (g1,) = pkg.interpret(m, {"a": a, "b": b}, gemm_path=3)
    (g2,) = pkg.interpret(m, {"a": a, "b": b}, gemm_path=3)
    np.testing.assert_array_equal(g1, g2)
    want = A.astype(np.float64) @ B.astype(np.float64)
    assert O.relative_error(g1, want) < TOL
    monkeypatch.setenv("SPX_H3_SPLITK", "0")
    (g0,) = pkg.interpret(m, {"a": a, "b": b}, gemm_path=3)
    assert O.relative_error(g0, want) < TOL


@pytest.mark.parametrize("shape", [(512, 131072, 256), (256, 32768, 512), (128, 65536, 256)],
                         ids=lambda s: "x".join(map(str, s)))
def test_gemm_h3_longk_weight_gradient(shape, monkeypatch):
    """SPX_H3_LONGK=1: few-tile long-K weight-gradient GEMMs (act^T @ dy,
    K = N*H*W) take the 3xFP16 kernel with in-kernel split-K (plan.py
    _h3_splitk; more than 4 splits fold from global memory): record path 3,
    within 1e-5 of float64, bit-identical across runs."""
    monkeypatch.setenv("SPX_H3_LONGK", "1")
    pkg = _pkg()
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.evaluator import last_executable
    M, K, N = shape
    rng = np.random.default_rng(9)
    a = rng.standard_normal((K, M)).astype(np.float32)
    b = rng.standard_normal((K, N)).astype(np.float32)
    m = _mm_module(M, K, N, True, False)
    (g1,) = pkg.interpret(m, {"a": a, "b": b})
    ex = last_executable()
    paths = [ex.plan.record_info(i)[1] for i, (k, _) in enumerate(ex.records()) if k == R.K_GEMM]
    assert paths == [3], paths
    (g2,) = pkg.interpret(m, {"a": a, "b": b})
    np.testing.assert_array_equal(g1, g2)
    want = a.T.astype(np.float64) @ b.astype(np.float64)
    assert np.all(np.isfinite(g1))
    assert O.relative_error(g1, want) < TOL


@pytest.mark.parametrize("at,bt", [(False, False), (True, True)])
@pytest.mark.parametrize("bn", ["128", "256"])
def test_gemm_h3_dynamic_range(at, bt, bn, monkeypatch):
    """Per-block scales: 128 x 128 blocks spanning 2^-40 .. 2^40, zero blocks,
    tiny and huge rows -- still <= 1e-5 against float64, per output block too."""
    monkeypatch.setenv("SPX_H3_BN", bn)
    pkg = _pkg()
    M, K, N = 512, 768, 384
    rng = np.random.default_rng(11)
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    for i in range(M // 128):
        for k in range(K // 128):
            A[i * 128:(i + 1) * 128, k * 128:(k + 1) * 128] *= 2.0 ** rng.integers(-40, 40)
    A[128:256, 256:384] = 0.0
    B[:, 5] *= 2.0 ** -30
    B[7, :] *= 2.0 ** 30
    A = A.astype(np.float32)
    B = B.astype(np.float32)
    a = np.ascontiguousarray(A.T) if at else A
    b = np.ascontiguousarray(B.T) if bt else B
    (got,) = pkg.interpret(_mm_module(M, K, N, at, bt), {"a": a, "b": b}, gemm_path=3)
    want = A.astype(np.float64) @ B.astype(np.float64)
    assert np.all(np.isfinite(got))
    assert O.relative_error(got, want) < TOL
    # accuracy does not hinge on the global maximum: every output row block on its own
    for i in range(M // 128):
        sl = slice(i * 128, (i + 1) * 128)
        assert O.relative_error(got[sl], want[sl]) < TOL, i


@pytest.mark.parametrize("shape", [(5, 7, 3), (64, 48, 80), (130, 70, 200), (256, 512, 384)])
def test_gemm_simt(shape):
    pkg = _pkg()
    M, K, N = shape
    rng = np.random.default_rng(2)
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((K, N)).astype(np.float32)
    (got,) = pkg.interpret(_mm_module(M, K, N), {"a": a, "b": b}, gemm_path=2)
    assert O.relative_error(got, a.astype(np.float64) @ b) < TOL


def test_elementwise_bitexact_large():
    """Fused add/mul/neg chains are bit-exact vs numpy at HBM-scale sizes."""
    pkg = _pkg()
    text = """func @main(%p: tensor<2048x4096xf32>, %m: tensor<2048x4096xf32>, %g: tensor<2048x4096xf32>, %b: tensor<4096xf32>) -> (tensor<2048x4096xf32>, tensor<2048x4096xf32>, tensor<2048x4096xf32>) {
  %c1 = constant 0.9 : tensor<2048x4096xf32>
  %a = mul %c1, %m : tensor<2048x4096xf32>
  %new_m = add %a, %g : tensor<2048x4096xf32>
  %c2 = constant 0.01 : tensor<2048x4096xf32>
  %s = mul %c2, %new_m : tensor<2048x4096xf32>
  %n = neg %s : tensor<2048x4096xf32>
  %new_p = add %p, %n : tensor<2048x4096xf32>
  %bb = broadcast %b {dims = [1]} : tensor<2048x4096xf32>
  %z = add %g, %bb : tensor<2048x4096xf32>
  %sq = mul %z, %z : tensor<2048x4096xf32>
  return %new_p, %new_m, %sq
}
"""
    m = pkg.parse_module(text)
    rng = np.random.default_rng(0)
    ins = {n: rng.standard_normal(t.dims).astype(np.float32) for n, t in m.func("main").args}
    got = pkg.interpret(m, ins)
    want = O.interpret(m, ins)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)


@pytest.mark.parametrize("dims,red", [((2048, 1024), [0]), ((2048, 1024), [0, 1]), ((2048, 1024), [1]),
                                      ((16, 64, 32), [0, 2]), ((8, 8, 8, 16), [1, 3])])
def test_reduce_large(dims, red):
    pkg = _pkg()
    t = "x".join(map(str, dims))
    kept = [d for i, d in enumerate(dims) if i not in red]
    rt = "tensor<" + "x".join(map(str, kept)) + ("x" if kept else "") + "f32>"
    text = (f"func @main(%x: tensor<{t}xf32>) -> {rt} {{\n"
            f"  %sq = mul %x, %x : tensor<{t}xf32>\n"
            f"  %r = reduce %sq {{dims = {red}}} : {rt}\n  return %r\n}}\n")
    m = pkg.parse_module(text)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(dims).astype(np.float32)
    (got,) = pkg.interpret(m, {"x": x})
    want = np.sum(x.astype(np.float64) ** 2, axis=tuple(red))
    assert O.relative_error(got, want) < TOL


def test_launch_counts_and_graph_replay():
    """A compiled plan replays as one CUDA graph and reproduces the eager run."""
    pkg = _pkg()
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.evaluator import default_device
    case = next(c for c in CASES if c["key"] == "step_tf2_bpmp_B2M2")
    m = pkg.parse_module(case["local_ir"])
    spec = pkg.ShardingSpec.from_json(case["sharding"])
    base = pkg.parse_module(case["dense_ir"])
    ins = case_inputs(case, base, 0)
    from paper_2401_11202_b200.evaluator import _chunk_slices
    mesh = m.mesh
    f = m.func("main")
    per = [{n: ins[n][_chunk_slices(ins[n].shape, spec.args[n], mesh, c)] for n, _ in f.args}
           for c in mesh.coords()]
    ex = Executable(m, device=default_device())
    ex.upload_args(per)
    ex.run()
    eager = ex.download_results()
    n_eager = ex.plan.launch_count()
    ex.plan.capture()
    ex.plan.replay()
    ex.device.sync()
    replay = ex.download_results()
    ex.close()
    assert n_eager > 0
    for a, b in zip(eager, replay):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("static,jit", [("1", "1"), ("0", "1"), ("0", "0")])
def test_elementwise_static_catalog_bitexact(static, jit, monkeypatch):
    """The compile-time-specialised kernels (ew_static.cu), the run-time
    specialised ones (ew_jit.cu) and the generic interpreter (ew.cu) all
    reproduce numpy bit-for-bit on the model zoo's programs (momentum update,
    square, square-grad, add, scale, sub)."""
    monkeypatch.setenv("SPX_EW_STATIC", static)
    monkeypatch.setenv("SPX_EW_JIT", jit)
    pkg = _pkg()
    text = """func @main(%p: tensor<512x1024xf32>, %m: tensor<512x1024xf32>, %g: tensor<512x1024xf32>, %z: tensor<512x1024xf32>) -> (tensor<512x1024xf32>, tensor<512x1024xf32>, tensor<512x1024xf32>, tensor<512x1024xf32>, tensor<512x1024xf32>, tensor<512x1024xf32>) {
  %c1 = constant 0.9 : tensor<512x1024xf32>
  %a = mul %c1, %m : tensor<512x1024xf32>
  %new_m = add %a, %g : tensor<512x1024xf32>
  %c2 = constant 0.01 : tensor<512x1024xf32>
  %s = mul %c2, %new_m : tensor<512x1024xf32>
  %n = neg %s : tensor<512x1024xf32>
  %new_p = add %p, %n : tensor<512x1024xf32>
  %sq = mul %z, %z : tensor<512x1024xf32>
  %two = constant 2.0 : tensor<512x1024xf32>
  %tz = mul %two, %z : tensor<512x1024xf32>
  %gr = mul %g, %tz : tensor<512x1024xf32>
  %ad = add %g, %z : tensor<512x1024xf32>
  %ng = neg %z : tensor<512x1024xf32>
  %sb = add %p, %ng : tensor<512x1024xf32>
  return %new_p, %new_m, %sq, %gr, %ad, %sb
}
"""
    m = pkg.parse_module(text)
    rng = np.random.default_rng(5)
    ins = {n: rng.standard_normal(t.dims).astype(np.float32) for n, t in m.func("main").args}
    got = pkg.interpret(m, ins)
    want = O.interpret(m, ins)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)


@pytest.mark.parametrize("epi", [1, 2, 3, 4])
def test_gemm_fused_epilogue_bitexact(epi, monkeypatch):
    """A GEMM with its elementwise consumer fused into the epilogue gives
    bit-identical results to the GEMM followed by the separate elementwise
    kernel (same accumulation, same IEEE ops), and matches the oracle."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_plan_cpu import EPILOGUE_PROGRAMS
    pkg = _pkg()
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.executable import Executable
    m = pkg.parse_module(EPILOGUE_PROGRAMS[epi])
    monkeypatch.setenv("SPX_EPILOGUE", "1")
    ex = Executable(m, devices=[0], dry=True)
    assert [p.epi for k, p in ex.records() if k == R.K_GEMM] == [epi]
    rng = np.random.default_rng(epi)
    ins = {n: rng.standard_normal(t.dims).astype(np.float32) for n, t in m.func("main").args}
    monkeypatch.setenv("SPX_EPILOGUE", "1")
    fused = pkg.interpret(m, ins)
    monkeypatch.setenv("SPX_EPILOGUE", "0")
    plain = pkg.interpret(m, ins, gemm_path=1)     # the fused epilogues live on the 3xTF32 kernel
    want = O.interpret(m, ins)
    for f, p, w in zip(fused, plain, want):
        np.testing.assert_array_equal(f, p)
        assert np.all(np.isfinite(f)) and O.relative_error(f, w) < TOL


def test_session_feed_pipeline():
    """Session.feed stages the next batch on a copy stream; step() consumes it
    in order -- results equal loading the same batch synchronously."""
    pkg = _pkg()
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.session import Session
    text = """func @main(%x: tensor<256x512xf32>, %w: tensor<512x256xf32>) -> tensor<256x256xf32> {
  %c = matmul %x, %w : tensor<256x256xf32>
  %o = add %c, %c : tensor<256x256xf32>
  return %o
}
"""
    m = pkg.parse_module(text)
    rng = np.random.default_rng(3)
    w = rng.standard_normal((512, 256)).astype(np.float32)
    xs = [rng.standard_normal((256, 512)).astype(np.float32) for _ in range(3)]
    sess = Session(m)
    sess.load({"x": xs[0], "w": w})
    sess.capture()
    dev = sess.device
    pins = []
    for x in xs:
        p = dev.pinned(x.shape)
        p[...] = x
        pins.append(p)
    sess.feed({"x": pins[0]})
    got = []
    for i in range(3):
        if i + 1 < 3:
            sess.feed({"x": pins[i + 1]})
        sess.step()
        sess.sync()
        got.append(sess.results()[0][0].copy())
    for x, g in zip(xs, got):
        want = O.interpret(m, {"x": x, "w": w})[0]
        assert O.relative_error(g, want) < TOL
    sess.close()


@pytest.mark.parametrize("M,N,K", [(1024, 512, 1024), (1024, 1024, 512), (1536, 512, 1024), (2048, 512, 640), (1024, 320, 1024)])
def test_gemm_inkernel_splitk(M, N, K, monkeypatch):
    """Critical-path GEMMs with few tiles split K inside the kernel (split-0
    CTAs fold the other splits' partials in split order): matches the oracle,
    and is bit-reproducible run to run (graph replays included)."""
    pkg = _pkg()
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.session import Session
    monkeypatch.setenv("SPX_SPLITK_INKERNEL", "1")
    text = f"""func @main(%x: tensor<{M}x{K}xf32>, %w: tensor<{K}x{N}xf32>) -> tensor<{M}x{N}xf32> {{
  %c = matmul %x, %w : tensor<{M}x{N}xf32>
  return %c
}}
"""
    m = pkg.parse_module(text)
    ex = Executable(m, devices=[0], dry=True)
    (k, p), = [r for r in ex.records() if r[0] == R.K_GEMM]
    assert p.sk_mode == 1 and p.splits > 1
    rng = np.random.default_rng(M + N + K)
    ins = {"x": rng.standard_normal((M, K)).astype(np.float32),
           "w": rng.standard_normal((K, N)).astype(np.float32)}
    want = O.interpret(m, ins)[0]
    sess = Session(m)
    sess.load(ins)
    sess.run()
    sess.sync()
    a = sess.results()[0][0].copy()
    sess.capture()
    for _ in range(3):
        sess.step()
    sess.sync()
    b = sess.results()[0][0]
    sess.close()
    assert np.all(np.isfinite(a)) and O.relative_error(a, want) < TOL
    np.testing.assert_array_equal(a, b)


@requires_gpu
@pytest.mark.gpu
def test_split_batch_bitexact(monkeypatch):
    """Consecutive standalone operand splits (here the hoisted splits of the
    batch and three weights, ragged sizes) run as one split_h16_batch_kernel
    launch; the GEMM results are bit-identical to one launch per split and
    within the fp32 bar of the oracle."""
    pkg = _pkg()
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.session import Session
    text = """func @main(%x: tensor<1024x520xf32>, %w1: tensor<520x384xf32>, %w2: tensor<384x640xf32>, %w3: tensor<640x328xf32>) -> tensor<1024x328xf32> {
  %h1 = matmul %x, %w1 : tensor<1024x384xf32>
  %h2 = matmul %h1, %w2 : tensor<1024x640xf32>
  %h3 = matmul %h2, %w3 : tensor<1024x328xf32>
  return %h3
}
"""
    m = pkg.parse_module(text)
    rng = np.random.default_rng(7)
    ins = {"x": rng.standard_normal((1024, 520)).astype(np.float32),
           "w1": (rng.standard_normal((520, 384)) * 1e-3).astype(np.float32),
           "w2": (rng.standard_normal((384, 640)) * 30).astype(np.float32),
           "w3": rng.standard_normal((640, 328)).astype(np.float32)}
    monkeypatch.setenv("SPX_SPLITK_F", "100000")      # no split-K: every GEMM on the 3xFP16 path
    monkeypatch.setenv("SPX_SPLIT_BATCH_FIRST", "0")  # one batch
    outs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("SPX_SPLIT_BATCH", mode)
        sess = Session(m)
        sess.load(ins)
        sess.capture()
        paths = [sess.ex.plan.record_info(i)[1] for i, (k, _) in enumerate(sess.ex._records) if k == R.K_SPLIT]
        if mode == "1":
            assert 2 in paths and paths.count(-2) >= 3, paths
        else:
            assert 2 not in paths and -2 not in paths, paths
        sess.step()
        sess.sync()
        outs[mode] = sess.results()[0][0].copy()
        sess.close()
    assert np.all(np.isfinite(outs["1"]))
    np.testing.assert_array_equal(outs["1"], outs["0"])
    want = O.interpret(m, ins)[0]
    assert O.relative_error(outs["1"], want) < TOL


@requires_gpu
@pytest.mark.gpu
@pytest.mark.parametrize("nbytes", [4, 4 << 20, (32 << 20) + 12, (200 << 20) + 4096 + 8])
def test_staged_copies_roundtrip(nbytes):
    """Pageable host <-> device through the pinned staging ring (spx_h2d_staged /
    spx_d2h_staged): bit-exact round trip for sizes below, at and across chunks."""
    from paper_2401_11202_b200 import runtime as R
    dev = R.Device(0)
    a = np.random.default_rng(nbytes % 97).integers(0, 2**31, nbytes // 4, dtype=np.int64).astype(np.uint32)
    d = dev.malloc(max(a.nbytes, 4))
    dev.h2d_staged(d, a)
    b = np.empty_like(a)
    dev.d2h_staged(b, d)
    np.testing.assert_array_equal(a, b)
    dev.free(d)


@requires_gpu
@pytest.mark.gpu
def test_h3_range_detection(monkeypatch):
    """A 128 x 128 operand block whose maximum lies outside [2^-45, 2^75] is
    reported (the fp16 split clamps its scale and its small elements lose
    precision) -- a warning by default, an error with SPX_STRICT_RANGE=1;
    in-range data raise nothing."""
    import warnings
    pkg = _pkg()
    from paper_2401_11202_b200 import runtime as R
    mm = pkg.parse_module("func @main(%a: tensor<256x256xf32>, %b: tensor<256x256xf32>) -> tensor<256x256xf32> {\n"
                          "  %c = matmul %a, %b : tensor<256x256xf32>\n  return %c\n}\n")
    rng = np.random.default_rng(5)
    a = rng.standard_normal((256, 256)).astype(np.float32)
    b = rng.standard_normal((256, 256)).astype(np.float32)
    R.h3_range_events(reset=True)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        pkg.interpret(mm, {"a": a, "b": b})               # in range: no warning
    a2 = a.copy()
    a2[:128, :128] *= np.float32(2.0 ** 90)
    with pytest.warns(RuntimeWarning, match="outside"):
        pkg.interpret(mm, {"a": a2, "b": b})
    monkeypatch.setenv("SPX_STRICT_RANGE", "1")
    with pytest.raises(FloatingPointError):
        pkg.interpret(mm, {"a": a2, "b": b})


JIT_PROGRAMS = {
    # nearest 2x2 upsample (the U-Net analog's rank-5 broadcast) times a full tensor
    "upsample": """func @main(%x: tensor<64x16x32xf32>, %y: tensor<64x2x16x2x32xf32>) -> tensor<64x2x16x2x32xf32> {
  %u = broadcast %x {dims = [0, 2, 4]} : tensor<64x2x16x2x32xf32>
  %p = mul %u, %y : tensor<64x2x16x2x32xf32>
  return %p
}
""",
    # a 3-D transpose (no float4 path) into exp and an add
    "transpose_exp": """func @main(%x: tensor<32x48x64xf32>, %z: tensor<64x32x48xf32>) -> tensor<64x32x48xf32> {
  %t = transpose %x {perm = [2, 0, 1]} : tensor<64x32x48xf32>
  %e = exp %t : tensor<64x32x48xf32>
  %s = add %e, %z : tensor<64x32x48xf32>
  return %s
}
""",
    # -(a) * b and a three-input chain, flat (the U-Net analog's gradient products)
    "neg_mul": """func @main(%a: tensor<1048576xf32>, %b: tensor<1048576xf32>, %c: tensor<1048576xf32>) -> (tensor<1048576xf32>, tensor<1048576xf32>) {
  %n = neg %a : tensor<1048576xf32>
  %p = mul %n, %b : tensor<1048576xf32>
  %q = mul %a, %b : tensor<1048576xf32>
  %k = constant 0.25 : tensor<1048576xf32>
  %r = mul %k, %c : tensor<1048576xf32>
  %s = mul %q, %r : tensor<1048576xf32>
  return %p, %s
}
""",
    # odd sizes (scalar path), row and column broadcasts, two outputs of one fused program
    "ragged_bcast": """func @main(%x: tensor<33x17xf32>, %r: tensor<17xf32>, %c: tensor<33xf32>) -> (tensor<33x17xf32>, tensor<33x17xf32>) {
  %rb = broadcast %r {dims = [1]} : tensor<33x17xf32>
  %cb = broadcast %c {dims = [0]} : tensor<33x17xf32>
  %a = add %x, %rb : tensor<33x17xf32>
  %m = mul %a, %cb : tensor<33x17xf32>
  %n = neg %m : tensor<33x17xf32>
  %o = add %n, %x : tensor<33x17xf32>
  return %m, %o
}
""",
}


@pytest.mark.parametrize("name", sorted(JIT_PROGRAMS))
def test_ew_jit_bitexact(name, monkeypatch):
    """Records outside the static catalog run as NVRTC-compiled kernels
    (record path -3) and match the interpreter bit-for-bit and numpy
    bit-for-bit (programs with exp: within the 1e-5 bar, as the golden
    `op_exp` cases)."""
    pkg = _pkg()
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.evaluator import last_executable
    m = pkg.parse_module(JIT_PROGRAMS[name])
    rng = np.random.default_rng(11)
    ins = {n: rng.standard_normal(t.dims).astype(np.float32) for n, t in m.func("main").args}
    monkeypatch.setenv("SPX_EW_JIT", "1")
    got = pkg.interpret(m, ins)
    ex = last_executable()
    paths = [ex.plan.record_info(i)[1] for i, (k, _) in enumerate(ex.records()) if k == R.K_EW]
    assert -3 in paths, paths
    monkeypatch.setenv("SPX_EW_JIT", "0")
    interp = pkg.interpret(m, ins)
    want = O.interpret(m, ins)
    for g, i, w in zip(got, interp, want):
        assert np.isfinite(g).all()
        np.testing.assert_array_equal(g, i, err_msg="jit vs interpreter")
        if name == "transpose_exp":
            # exp then add: CUDA's expf and numpy's differ in the last ulp, which
            # the add can expose where e^x and z cancel -> the exp bar (1e-5)
            assert O.relative_error(g, w) < TOL
        else:
            np.testing.assert_array_equal(g, w)


UPSAMPLE_MM = """func @main(%x: tensor<256x16x128xf32>, %w: tensor<128x256xf32>) -> tensor<16384x256xf32> {
  %u = broadcast %x {dims = [0, 2, 4]} : tensor<256x2x16x2x128xf32>
  %r = reshape %u {dims = [16384, 128]} : tensor<16384x128xf32>
  %c = matmul %r, %w : tensor<16384x256xf32>
  return %c
}
"""


@pytest.mark.parametrize("pieces_only", ["1", "0"])
def test_ew_jit_fused_split_bitexact(pieces_only, monkeypatch):
    """A run-time specialised elementwise record (the U-Net analog's upsample
    broadcast) whose output feeds a 3xFP16 GEMM emits the GEMM's fp16 pieces
    itself (split record path -1): the GEMM result is bit-identical to the
    standalone split's, with the fp32 output skipped (read only through its
    pieces) or stored (SPX_PIECES_ONLY=0)."""
    pkg = _pkg()
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.evaluator import last_executable
    monkeypatch.setenv("SPX_OVERLAP", "0")       # one stream: the split right after its producer
    monkeypatch.setenv("SPX_PIECES_ONLY", pieces_only)
    m = pkg.parse_module(UPSAMPLE_MM)
    rng = np.random.default_rng(4)
    ins = {"x": rng.standard_normal((256, 16, 128)).astype(np.float32),
           "w": rng.standard_normal((128, 256)).astype(np.float32)}
    monkeypatch.setenv("SPX_EW_JIT_SPLIT", "1")
    fused = pkg.interpret(m, ins)
    ex = last_executable()
    info = [ex.plan.record_info(i) for i in range(len(ex.records()))]
    assert any(k == R.K_EW and p == -3 for k, p in info), info
    assert any(k == R.K_SPLIT and p == -1 for k, p in info), info
    monkeypatch.setenv("SPX_EW_JIT_SPLIT", "0")
    plain = pkg.interpret(m, ins)
    np.testing.assert_array_equal(fused[0], plain[0])
    want = O.interpret(m, ins)
    assert O.relative_error(fused[0], want[0]) < TOL
