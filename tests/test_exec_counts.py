"""Executed work vs the reference simulator's prediction (CPU: derived from
the records exactly as the runtime counts them, runtime.cu tally_record /
record_flops; the GPU tests read the runtime's own counters).

* collectives: every IR collective the program lists
  (`collective_counts`, spmd.py:264-271) is either issued by exactly one
  record or served by an identical earlier collective of the same immutable
  buffer (CSE); with SPX_COLL_CSE=0 every one is issued, so the executed
  counts equal the simulator's;
* FLOPs (`simulate().compute_flops`, sim.py:86-100, :209-229): the kernels
  issue exactly the simulator's FLOPs minus the elementwise ops the compiler
  folds at build time (constant operands only).
"""
import pytest

from conftest import golden_cases
from record_sim import _dry_comms
from paper_2401_11202_b200.evaluator import _Dense
from paper_2401_11202_b200.executable import Executable
from paper_2401_11202_b200.ir import collective_counts, compute_flops, parse_module
from paper_2401_11202_b200.programs import load_program

CASES = [c for c in golden_cases() if "local_ir" in c and c.get("error") is None]
CONFIG_PROGRAMS = ["c1_mlp_bp_B2", "c2_tf1_bpmp_B2M4", "c2_tf8_bpmp_B2M4", "c3_tf1_bpz3_B8",
                   "c4_unet_bpz2_B8", "c5_tf1_bpmpz3emb_B2M2E2", "c5_tf8_bpmpz3emb_B2M2E2"]


def _check(module, ex, exact):
    w = ex.work_report()
    prog = collective_counts(module)
    assert w["collectives"]["program"] == prog
    for k, n in prog.items():
        assert w["collectives"]["executed"][k] + w["collectives"]["cse_elided"][k] == n, (k, w)
        if exact:
            assert w["collectives"]["executed"][k] == n, (k, w)
    sim = compute_flops(module)
    assert w["flops"]["simulator"] == sim
    assert w["flops"]["executed"] + w["flops"]["folded"] == pytest.approx(sim, rel=1e-12, abs=1e-6), w


@pytest.mark.parametrize("cse", ["1", "0"])
@pytest.mark.parametrize("mode", ["local", "nccl"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c["key"])
def test_golden_executed_work(case, mode, cse, monkeypatch):
    monkeypatch.setenv("SPX_COLL_CSE", cse)
    m = parse_module(case["local_ir"])
    if mode == "local":
        ex = Executable(m, dry=True)
    else:
        ex = Executable(m, devices=[0], comm_mode="nccl", dry=True, comm_factory=lambda e: _dry_comms(e, True))
    _check(m, ex, exact=(cse == "0"))


@pytest.mark.parametrize("case", [c for c in golden_cases() if "dense_ir" in c], ids=lambda c: c["key"])
def test_dense_executed_flops(case):
    m = parse_module(case["dense_ir"])
    ex = Executable(_Dense(m), devices=[0], dry=True)
    _check(m, ex, exact=True)


@pytest.mark.parametrize("cse", ["1", "0"])
@pytest.mark.parametrize("mode", ["local", "nccl"])
@pytest.mark.parametrize("name", CONFIG_PROGRAMS)
def test_config_executed_work(name, mode, cse, monkeypatch):
    monkeypatch.setenv("SPX_COLL_CSE", cse)
    p = load_program(name)
    if mode == "local":
        ex = Executable(p.local, dry=True)
    else:
        ex = Executable(p.local, devices=[0], comm_mode="nccl", dry=True, comm_factory=lambda e: _dry_comms(e, True))
    _check(p.local, ex, exact=(cse == "0"))
    assert ex.work_report()["collectives"]["program"] == p.meta["counts"]      # the partitioner's own export
    assert ex.comp.flops == p.meta["cost"]["compute_flops"]                     # simulate(...).compute_flops


@pytest.mark.parametrize("name", CONFIG_PROGRAMS + ["c2_tf8_dense", "c4_unet_dense", "c3_tf2_dense"])
def test_fused_split_does_not_reuse_producer_inputs(name):
    """A split placed right after the elementwise kernel producing its source
    runs inside that kernel's launch (runtime.cu ew_static_split); its pieces
    must not occupy memory the producer still reads (liveness packing would
    otherwise recycle the producer's last-use inputs for them)."""
    from paper_2401_11202_b200.plan import _align
    p = load_program(name)
    m = p.dense if name.endswith("dense") else p.local
    ex = Executable(_Dense(m) if name.endswith("dense") else m, devices=[0] if name.endswith("dense") else None,
                    dry=True)
    c = ex.comp
    ks = c.kernels

    def iv(b):
        return ex.off[b], ex.off[b] + _align(c.buffers[b])
    n = 0
    for i, k in enumerate(ks):
        if k.kind == "split" and i and ks[i - 1].kind == "ew" and k.data["src"][0] in ks[i - 1].outs:
            n += 1
            p0, p1 = iv(k.outs[0])
            for b in ks[i - 1].ins:
                a0, a1 = iv(b)
                assert p1 <= a0 or a1 <= p0, (name, i, b)
    assert n > 0


@pytest.mark.parametrize("name", CONFIG_PROGRAMS + ["c2_tf8_dense", "c4_unet_dense", "c3_tf2_dense"])
def test_pieces_only_sources_have_only_piece_readers(name):
    """SPX_SPLIT_PIECES_ONLY lets the launch producing a split's source skip its
    fp32 store: valid only if every reader of that source is a block-scaled
    GEMM reading THIS split's pieces and the source is no function result."""
    p = load_program(name)
    dense = name.endswith("dense")
    ex = Executable(_Dense(p.dense) if dense else p.local, devices=[0] if dense else None, dry=True)
    ks = ex.comp.kernels
    results = set(ex.comp.result_bufs)
    n = 0
    for k in ks:
        if k.kind == "split" and k.data.get("pieces_only"):
            n += 1
            src, piece = k.data["src"][0], k.outs[0]
            assert src not in results
            for r in ks:
                if r is not k and src in r.ins:
                    assert r.kind == "gemm", (name, r.kind)
                    assert piece in (r.data.get("h3a"), r.data.get("h3b")), name
    if name.startswith(("c2", "c3", "c5")):
        assert n > 0
