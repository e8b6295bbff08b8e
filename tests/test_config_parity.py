"""GPU parity on the BASELINE configurations' own programs, default path.

The reference's release gate is a differential check of every schedule's
partitioned step (`test_acceptance.py:64-92`, `spindle verify`,
cli.py:121-160).  Here every BASELINE config's program -- its mesh, its
tactics, full width; transformer depth reduced to 1-2 identical blocks where
the CPU oracle cannot hold the full depth -- runs through the
drop-in `spmd_interpret` (all mesh devices on one B200) and, for the dense
1-GPU programs, `interpret`, with every performance knob at its default:
block-scaled 3xFP16 tcgen05 GEMMs on shared operand splits, splits fused into
the producing elementwise kernel, batched argument splits, four streams, PDL,
CUDA-graph replay from the compiled-plan cache.  Each call's outputs are
compared with the oracle restatement of the reference evaluator on the same
inputs: all finite, `relative_error` < 1e-5 (spmd_interp.py:25-31).
The plan is checked to have actually used those kernels (record paths).
"""
import numpy as np
import pytest

from conftest import TOL, requires_gpu
from oracle import spmd_oracle as O

pytestmark = [pytest.mark.gpu, requires_gpu]

# (program, mode, input scale, seeds): scale per SURVEY §8(d)
CONFIGS = [
    ("c1_mlp_bp_B2", "spmd", 0.25, [0, 1]),          # C1 in full: mlp b=256 d=1024, BP on B:2
    ("c1_mlp_dense", "dense", 0.25, [0]),
    ("c2_tf1_bpmp_B2M4", "spmd", 0.02, [0, 1]),      # C2: BP+MP on 2x4, d=1024 d_ff=4096 b=2048
    ("c2_tf2_bpmp_B2M4", "spmd", 0.02, [0]),
    ("c2_tf8_dense", "dense", 0.02, [0]),             # C2 at full depth: the N=1 benchmark program
    ("c3_tf1_bpz3_B8", "spmd", 0.02, [0]),            # C3: BP+Z3 on B:8, d=2048 d_ff=8192 b=8192
    ("c3_tf2_dense", "dense", 0.02, [0]),
    ("c4_unet_bpz2_B8", "spmd", 0.05, [0]),           # C4: U-Net analog in full, BP+Z2 on B:8
    ("c4_unet_dense", "dense", 0.05, [0]),
    ("c5_tf1_bpmpz3emb_B2M2E2", "spmd", 0.02, [0, 1]),  # C5: BP+MP+Z3+EMB on 2x2x2
    ("c5_tf2_bpmpz3emb_B2M2E2", "spmd", 0.02, [0]),
]


def plan_paths(ex):
    """Which kernels the plan launches: GEMM paths (3 = block-scaled 3xFP16,
    1 = 3xTF32, 2 = SIMT), operand splits (-1 fused into the producing
    elementwise kernel, -2 inside a batched launch), static elementwise,
    run-time specialised elementwise (ew_jit.cu, path -3), interpreter."""
    from paper_2401_11202_b200 import runtime as R
    out = {"gemm": {}, "split": {}, "ew_static": 0, "ew_jit": 0, "ew_generic": 0}
    for i, (kind, _) in enumerate(ex.records()):
        k, path = ex.plan.record_info(i)
        if k == R.K_GEMM:
            out["gemm"][path] = out["gemm"].get(path, 0) + 1
        elif k == R.K_SPLIT:
            out["split"][path] = out["split"].get(path, 0) + 1
        elif k == R.K_EW:
            out["ew_static" if path > 0 else "ew_jit" if path == -3 else "ew_generic"] += 1
    return out


@pytest.mark.parametrize("name,mode,scale,seeds", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_config_program_parity(name, mode, scale, seeds):
    import paper_2401_11202_b200 as pkg
    from paper_2401_11202_b200.evaluator import last_executable
    prog = pkg.load_program(name)
    for s in seeds:
        ins = pkg.programs.synthetic_inputs(prog.dense, seed=s, scale=scale)
        if mode == "spmd":
            want = O.spmd_interpret(prog.local, prog.sharding, ins)
            runs = [pkg.spmd_interpret(prog.local, prog.sharding, ins) for _ in range(2)]
        else:
            want = O.interpret(prog.dense, ins)
            runs = [pkg.interpret(prog.dense, ins) for _ in range(2)]
        # first call: eager launch of the compiled plan; second: CUDA-graph replay from the cache
        for got in runs:
            assert len(got) == len(want)
            for j, (g, w) in enumerate(zip(got, want)):
                assert g.shape == w.shape and g.dtype == w.dtype, j
                assert np.all(np.isfinite(g)), f"{name} output {j} not finite"
                err = O.relative_error(g, w)
                assert err < TOL, f"{name} seed {s} output {j}: relative error {err:.3e}"
        for a, b in zip(runs[0], runs[1]):
            np.testing.assert_array_equal(a, b)          # graph replay == eager, bit for bit
    ex = last_executable()
    _check_executed_work(prog.local if mode == "spmd" else prog.dense, ex, exact=False)
    paths = plan_paths(ex)
    n_gemm = sum(paths["gemm"].values())
    assert n_gemm > 0
    # every GEMM on a tcgen05 path: block-scaled 3xFP16 (3) by default, the
    # 3xTF32 split-K kernel (1) for few-tile long-K weight gradients; none on SIMT
    assert paths["gemm"].get(2, 0) == 0, paths
    assert paths["gemm"].get(3, 0) >= 1, paths
    assert paths["ew_static"] > 0, paths
    assert paths["ew_generic"] == 0, paths               # the rest run as NVRTC-compiled kernels
    if not name.startswith("c1"):
        assert paths["split"].get(-1, 0) > 0, paths      # elementwise kernels emit the fp16 pieces


def _check_executed_work(module, ex, exact):
    """The runtime's own counters (spx_plan_exec_stats) against the reference
    simulator: executed + CSE-elided collectives = collective_counts
    (spmd.py:264-271), executed + compile-time-folded FLOPs =
    simulate().compute_flops (sim.py:209-229)."""
    import paper_2401_11202_b200 as pkg
    w = ex.work_report()
    assert w["collectives"]["source"].startswith("runtime counters"), w
    pred = ex.issued_per_run()
    assert w["collectives"]["executed"] == pred["coll"], (w, pred)     # counters == records
    assert w["flops"]["executed"] * ex.ndev == pytest.approx(pred["flops"], rel=1e-12)
    prog = pkg.collective_counts(module)
    for k, n in prog.items():
        assert w["collectives"]["executed"][k] + w["collectives"]["cse_elided"][k] == n, (k, w)
        if exact:
            assert w["collectives"]["executed"][k] == n, (k, w)
    sim = pkg.compute_flops(module)
    assert w["flops"]["executed"] + w["flops"]["folded"] == pytest.approx(sim, rel=1e-12), w


@pytest.mark.parametrize("name", ["c5_tf1_bpmpz3emb_B2M2E2", "c3_tf1_bpz3_B8"])
def test_count_exact_mode(name, monkeypatch):
    """SPX_COLL_CSE=0: every collective the program lists is issued -- the
    executed counts equal the simulator's -- and the results still match."""
    import paper_2401_11202_b200 as pkg
    from paper_2401_11202_b200.evaluator import last_executable
    monkeypatch.setenv("SPX_COLL_CSE", "0")
    prog = pkg.load_program(name)
    ins = pkg.programs.synthetic_inputs(prog.dense, seed=3, scale=0.02)
    got = pkg.spmd_interpret(prog.local, prog.sharding, ins)
    want = O.spmd_interpret(prog.local, prog.sharding, ins)
    for g, w in zip(got, want):
        assert np.all(np.isfinite(g)) and O.relative_error(g, w) < TOL
    _check_executed_work(prog.local, last_executable(), exact=True)


def test_smoke_entry():
    """`__graft_entry__.smoke()` -- C1 at its stated size through the default path."""
    import __graft_entry__
    __graft_entry__.smoke()


def _host_ram_gb():
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 0.0


@pytest.mark.skipif(_host_ram_gb() < 120, reason="the CPU oracle needs ~90 GB of host RAM at C3's full size")
def test_c3_full_size_parity():
    """The N=1 benchmark program itself -- C3 at 32 blocks, d_model 2048,
    d_ff 8192, batch 8192 -- through `interpret` on the default path, against
    the oracle's dense `interpret` on the host (~1 min): every one of the 258
    outputs finite and within 1e-5 (profiles/r02_c3_full_parity.txt)."""
    import paper_2401_11202_b200 as pkg
    prog = pkg.load_program("c3_tf32_dense")
    ins = pkg.programs.synthetic_inputs(prog.dense, seed=0, scale=0.02)
    got = pkg.interpret(prog.dense, ins)
    want = O.interpret(prog.dense, ins)
    assert len(got) == len(want) == 258
    for j, (g, w) in enumerate(zip(got, want)):
        assert np.all(np.isfinite(g)), j
        assert O.relative_error(g, w) < TOL, (j, O.relative_error(g, w))
