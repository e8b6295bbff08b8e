"""Plan compiler on CPU: lower every golden program to native records, execute
them with the record simulator, and compare with the reference's outputs.
Also checks the executed collective counts and FLOPs against the simulator
(`collective_counts`, spmd.py:264-271; `simulate().compute_flops`,
sim.py:209-229) as recorded in the golden cases."""
import numpy as np
import pytest

from conftest import TOL, case_expected, case_inputs, golden_cases
from oracle.spmd_oracle import DivergenceError as OracleDivergence
from paper_2401_11202_b200.evaluator import DivergenceError, relative_error
from paper_2401_11202_b200.ir import ShardingSpec, parse_module
from record_sim import sim_dense, sim_spmd

CASES = golden_cases()

# data movement / elementwise programs must be bit-exact (SURVEY §8c parity rules)
BITEXACT_GROUPS = ("rule",)


@pytest.mark.parametrize("case", [c for c in CASES if "local_ir" in c], ids=lambda c: c["key"])
def test_plan_spmd_sim(case):
    m = parse_module(case["local_ir"])
    spec = ShardingSpec.from_json(case["sharding"])
    base = parse_module(case["dense_ir"]) if "dense_ir" in case else m
    for s in case["seeds"]:
        ins = case_inputs(case, base, s)
        if case.get("error") == "DivergenceError":
            with pytest.raises(DivergenceError):
                sim_spmd(m, spec, ins)
            continue
        got, ex = sim_spmd(m, spec, ins)
        assert ex.comp.counts == case["counts"]
        if "compute_flops" in case:
            assert ex.comp.flops == case["compute_flops"]
        for g, w in zip(got, case_expected(case, s, "spmd")):
            assert np.all(np.isfinite(g))
            if case["group"] in BITEXACT_GROUPS and "exp" not in case["local_ir"]:
                np.testing.assert_array_equal(g, w)
            else:
                assert relative_error(g, w) < TOL


@pytest.mark.parametrize("case", [c for c in CASES if "dense_ir" in c], ids=lambda c: c["key"])
def test_plan_dense_sim(case):
    m = parse_module(case["dense_ir"])
    for s in case["seeds"]:
        ins = case_inputs(case, m, s)
        got, _ = sim_dense(m, ins)
        for g, w in zip(got, case_expected(case, s, "dense")):
            assert g.shape == w.shape
            assert relative_error(g, w) < TOL


def test_momentum_update_is_one_kernel():
    """m' = 0.9 m + g ; p' = p + -(0.01 m') fuses into one two-output kernel."""
    from paper_2401_11202_b200.executable import Executable
    text = """func @main(%p: tensor<64x64xf32>, %m: tensor<64x64xf32>, %g: tensor<64x64xf32>) -> (tensor<64x64xf32>, tensor<64x64xf32>) {
  %c1 = constant 0.9 : tensor<64x64xf32>
  %a = mul %c1, %m : tensor<64x64xf32>
  %new_m = add %a, %g : tensor<64x64xf32>
  %c2 = constant 0.01 : tensor<64x64xf32>
  %b = mul %c2, %new_m : tensor<64x64xf32>
  %n = neg %b : tensor<64x64xf32>
  %new_p = add %p, %n : tensor<64x64xf32>
  return %new_p, %new_m
}
"""
    m = parse_module(text)
    ex = Executable(m, devices=[0], dry=True)
    kinds = [k for k, _ in ex.records()]
    assert kinds == [1]                     # a single EW record
    (_, p), = ex.records()
    assert p.n_out == 2 and p.n_in == 3 and p.vec == 1
    rng = np.random.default_rng(0)
    ins = {n: rng.standard_normal((64, 64)).astype(np.float32) for n in ("p", "m", "g")}
    got, _ = sim_dense(m, ins)
    from oracle.spmd_oracle import interpret
    want = interpret(m, ins)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)


def test_split_k_gemm_sim(monkeypatch):
    """Few-tile GEMMs with long K split into partials + a deterministic
    reduction (the 3xTF32 form; by default such GEMMs take the 3xFP16
    kernel's in-kernel split, test_longk_weight_gradient_takes_h3_splitk)."""
    monkeypatch.setenv("SPX_H3_LONGK", "0")
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.executable import Executable
    text = """func @main(%a: tensor<4096x128xf32>, %b: tensor<4096x256xf32>) -> tensor<128x256xf32> {
  %at = transpose %a {perm = [1, 0]} : tensor<128x4096xf32>
  %c = matmul %at, %b : tensor<128x256xf32>
  return %c
}
"""
    m = parse_module(text)
    ex = Executable(m, devices=[0], dry=True)
    gem = [p for k, p in ex.records() if k == R.K_GEMM]
    assert gem[0].splits > 1 and gem[0].a_mn_major == 1
    assert [k for k, _ in ex.records()] == [R.K_GEMM, R.K_REDUCE]
    rng = np.random.default_rng(0)
    ins = {"a": rng.standard_normal((4096, 128)).astype(np.float32),
           "b": rng.standard_normal((4096, 256)).astype(np.float32)}
    got, _ = sim_dense(m, ins)
    assert relative_error(got[0], ins["a"].T.astype(np.float64) @ ins["b"]) < TOL


EPILOGUE_PROGRAMS = {
    # residual add: out = x + A.B
    1: """func @main(%a: tensor<256x128xf32>, %b: tensor<128x256xf32>, %x: tensor<256x256xf32>) -> tensor<256x256xf32> {
  %c = matmul %a, %b : tensor<256x256xf32>
  %o = add %x, %c : tensor<256x256xf32>
  return %o
}
""",
    # square activation, product kept for a later reader
    2: """func @main(%a: tensor<256x128xf32>, %b: tensor<128x256xf32>, %x: tensor<256x256xf32>) -> (tensor<256x256xf32>, tensor<256x256xf32>) {
  %c = matmul %a, %b : tensor<256x256xf32>
  %s = mul %c, %c : tensor<256x256xf32>
  %u = mul %c, %x : tensor<256x256xf32>
  return %s, %u
}
""",
    # backward of the square: g = A.B * (x * 2)
    3: """func @main(%a: tensor<256x128xf32>, %b: tensor<128x256xf32>, %x: tensor<256x256xf32>) -> tensor<256x256xf32> {
  %c = matmul %a, %b : tensor<256x256xf32>
  %k = constant 2.0 : tensor<256x256xf32>
  %x2 = mul %x, %k : tensor<256x256xf32>
  %o = mul %c, %x2 : tensor<256x256xf32>
  return %o
}
""",
    # momentum SGD on a weight gradient
    4: """func @main(%a: tensor<128x256xf32>, %b: tensor<128x256xf32>, %m: tensor<256x256xf32>, %p: tensor<256x256xf32>) -> (tensor<256x256xf32>, tensor<256x256xf32>) {
  %at = transpose %a {perm = [1, 0]} : tensor<256x128xf32>
  %g = matmul %at, %b : tensor<256x256xf32>
  %c1 = constant 0.9 : tensor<256x256xf32>
  %v = mul %c1, %m : tensor<256x256xf32>
  %nm = add %v, %g : tensor<256x256xf32>
  %c2 = constant 0.01 : tensor<256x256xf32>
  %w = mul %c2, %nm : tensor<256x256xf32>
  %n = neg %w : tensor<256x256xf32>
  %np = add %p, %n : tensor<256x256xf32>
  return %np, %nm
}
""",
}


@pytest.mark.parametrize("epi", sorted(EPILOGUE_PROGRAMS))
def test_gemm_epilogue_fusion_sim(epi, monkeypatch):
    """Each fused epilogue is recognised (no separate elementwise kernel for
    the GEMM's consumer) and the fused records reproduce the oracle."""
    from oracle.spmd_oracle import interpret
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.executable import Executable
    monkeypatch.setenv("SPX_EPILOGUE", "1")
    m = parse_module(EPILOGUE_PROGRAMS[epi])
    ex = Executable(m, devices=[0], dry=True)
    gem = [p for k, p in ex.records() if k == R.K_GEMM]
    assert len(gem) == 1 and gem[0].epi == epi
    rng = np.random.default_rng(epi)
    f = m.func("main")
    ins = {n: rng.standard_normal(t.dims).astype(np.float32) for n, t in f.args}
    got, _ = sim_dense(m, ins)
    want = interpret(m, ins)
    for g, w in zip(got, want):
        assert relative_error(g, w) < TOL


@pytest.mark.parametrize("name", ["c4_unet_bpz2_B4", "c2_tf8_bpmp_B2M2", "c2_tf8_bp_B2", "c3_tf32_bpz3_B8",
                                  "c5_tf8_bpmpz3emb_B2M2E2"])
def test_cross_rank_collectives_on_one_stream(name, monkeypatch):
    """Forward progress by construction: in NCCL mode every
    cross-rank collective (peer kernel or NCCL call) is issued on the single
    collective stream, in program order, so side-stream GEMMs are allowed at
    any rank count; the staging region of NCCL relayouts is part of every
    user's conflict set."""
    from record_sim import _dry_comms
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.programs import load_program
    for k in ("SPX_CONCURRENT_GEMM", "SPX_COLL_ONE_STREAM", "SPX_SIDE_ALL_COLLECTIVES"):
        monkeypatch.delenv(k, raising=False)
    p = load_program(name)
    ex = Executable(p.local, devices=[0], comm_mode="nccl", dry=True, comm_factory=lambda e: _dry_comms(e, True))
    streams = {(k.kind, ex.stream_of.get(i, 0)) for i, k in enumerate(ex.comp.kernels)}
    assert ("gemm", ex.COMPUTE) in streams, name
    for i, k in enumerate(ex.comp.kernels):
        if k.kind == "coll" and k.data["kind"] != "all_slice":
            assert ex.stream_of.get(i) == ex.COMM, (name, i, k.data["kind"])
    # every record that talks to another rank sits on the collective stream
    rec_stream = {}
    for idx, st, _ in ex.sched:
        rec_stream[idx] = st
    for idx, (kind, _) in enumerate(ex.records()):
        if kind in (R.K_NCCL, R.K_PEER):
            assert rec_stream.get(idx, 0) == ex.COMM, (name, idx)


@pytest.mark.parametrize("name", ["c1_mlp_dense", "c3_tf2_dense", "c5_tf1_bpmpz3emb_B2M2E2"])
def test_io_copies_in_the_plan(name):
    """io=True (the drop-in call): one H2D copy record per (argument, device)
    on the H2D stream, placed before the first record reading the argument,
    one D2H copy per (result, device) on the D2H stream after the record that
    last writes the result; every reader/writer ordering is a schedule edge."""
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.evaluator import _Dense
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.programs import load_program
    p = load_program(name)
    dense = p.local is None or name.endswith("dense")
    m = p.dense if dense else p.local
    ex = Executable(_Dense(m) if dense else m, devices=[0] if dense else None, dry=True, io=True)
    recs = ex.records()
    stream = {i: s for i, s, _ in ex.sched}
    nargs = len(ex.comp.arg_bufs) * ex.ndev
    nres = len(ex.comp.result_bufs) * ex.ndev
    assert len(ex.copy_in) == nargs and len(ex.copy_out) == nres
    for idx in ex.copy_in.values():
        assert recs[idx][0] == R.K_COPY and recs[idx][1].dir == 0 and stream[idx] == ex.H2D
    for idx in ex.copy_out.values():
        assert recs[idx][0] == R.K_COPY and recs[idx][1].dir == 1 and stream[idx] == ex.D2H
    # kernel order: each argument's copy precedes its readers, each result's copy follows its writers
    pos = {id(k): i for i, k in enumerate(ex.comp.kernels)}
    for i, k in enumerate(ex.comp.kernels):
        if k.kind == "copy" and k.data["dir"] == 0:
            assert all(i < j for j, r in enumerate(ex.comp.kernels) if k.data["buf"] in r.ins)
        if k.kind == "copy" and k.data["dir"] == 1:
            assert all(j < i for j, r in enumerate(ex.comp.kernels) if k.data["buf"] in r.outs)
    assert pos


def test_longk_weight_gradient_takes_h3_splitk(monkeypatch):
    """SPX_H3_LONGK=1: a few-tile long-K GEMM (act^T @ dy) is one 3xFP16
    record with an in-kernel split count (no workspace + reduce records); with
    the 3xFP16 kernel off it keeps the 3xTF32 workspace split-K and its
    reduction."""
    monkeypatch.setenv("SPX_H3_LONGK", "1")
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.executable import Executable
    from test_gpu_parity import _mm_module
    m = _mm_module(512, 131072, 256, True, False)
    ex = Executable(m, devices=[0], dry=True)
    g = [p for k, p in ex.records() if k == R.K_GEMM]
    assert len(g) == 1 and g[0].path == 3 and g[0].h3_splitk > 1 and g[0].h3_shared == 1
    assert not any(k == R.K_REDUCE for k, _ in ex.records())
    monkeypatch.setenv("SPX_GEMM_H3", "0")
    ex = Executable(m, devices=[0], dry=True)
    g = [p for k, p in ex.records() if k == R.K_GEMM]
    assert len(g) == 1 and g[0].splits > 1
    assert any(k == R.K_REDUCE for k, _ in ex.records())


@pytest.mark.parametrize("name", ["c2_tf8_bpmp_B2M2", "c3_tf2_bpz3_B4", "c5_tf1_bpmpz3emb_B2M2E2"])
def test_gradient_collectives_hoisted_and_critical_producers_on_main(name, monkeypatch):
    """Gradient collectives (outputs read only by the updates) follow their
    gradient instead of the whole backward pass; the kernel order stays a
    valid topological order; GEMMs whose output feeds a critical-path
    collective stay on the main stream (timelines in
    profiles/r02_timeline_n4.txt)."""
    from record_sim import _dry_comms
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.programs import load_program
    for k in ("SPX_HOIST_COLL", "SPX_CRIT_PRODUCERS_MAIN", "SPX_COLL_ONE_STREAM"):
        monkeypatch.delenv(k, raising=False)
    p = load_program(name)
    ex = Executable(p.local, devices=[0], comm_mode="nccl", dry=True, comm_factory=lambda e: _dry_comms(e, True))
    ks = ex.comp.kernels
    made = set(ex.comp.arg_bufs)
    for k in ks:                                      # topological
        assert all(b in made for b in k.ins), k
        made.update(k.outs)
    prod = {b: i for i, k in enumerate(ks) for b in k.outs}
    readers = {}
    for i, k in enumerate(ks):
        for b in k.ins:
            readers.setdefault(b, []).append(i)
    grad_colls = 0
    for i, k in enumerate(ks):
        if k.kind != "coll" or k.data["kind"] in ("all_slice",):
            continue
        rd = [j for b in k.outs for j in readers.get(b, [])]
        if rd and all(ex._terminal(ks[j]) or ks[j].kind == "coll" for j in rd):
            grad_colls += 1
            # hoisted: within a few kernels of its gradient
            src = max(prod[b] for b in k.ins if b in prod)
            assert i - src <= 16, (name, i, src)
        elif i not in ex.coll_offcrit:
            # a critical collective: its GEMM producers run on the main stream
            for b in k.ins:
                j = prod.get(b)
                if j is not None and ks[j].kind == "gemm":
                    assert ex.stream_of.get(j, 0) == 0, (name, i, j)
    assert grad_colls > 0
