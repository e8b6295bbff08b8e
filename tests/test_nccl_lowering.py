"""One-process-per-GPU lowering (NCCL mode), checked on CPU: every rank's
records run in lockstep through the record simulator with NCCL semantics, and
the reassembled results match the reference's golden outputs; plus the
multi-process host logic (communicator plan + unique-id exchange) over a real
world_size-2 gloo group."""
import os

import numpy as np
import pytest

from conftest import TOL, case_expected, case_inputs, golden_cases
from paper_2401_11202_b200.evaluator import DivergenceError, relative_error
from paper_2401_11202_b200.ir import ShardingSpec, parse_module
from record_sim import sim_nccl

CASES = [c for c in golden_cases() if "local_ir" in c]


@pytest.mark.parametrize("peer", [False, True, "ce"], ids=["nccl", "peer", "ce"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c["key"])
def test_nccl_mode_matches_reference(case, peer, monkeypatch):
    """'ce': the copy-engine all-gather and reduce-scatter at every size."""
    if peer == "ce":
        monkeypatch.setenv("SPX_CE_MIN_BYTES", "0")
        monkeypatch.setenv("SPX_CE_RS", "1")
        peer = True
    m = parse_module(case["local_ir"])
    spec = ShardingSpec.from_json(case["sharding"])
    base = parse_module(case["dense_ir"]) if "dense_ir" in case else m
    s = case["seeds"][0]
    ins = case_inputs(case, base, s)
    if case.get("error") == "DivergenceError":
        with pytest.raises(DivergenceError):
            sim_nccl(m, spec, ins, peer=peer)
        return
    got, exs = sim_nccl(m, spec, ins, peer=peer)
    assert exs[0].comp.counts == case["counts"]
    for g, w in zip(got, case_expected(case, s, "spmd")):
        assert relative_error(g, w) < TOL
    if peer:
        # the peer all-reduce folds in member order like the reference's
        # _combine: bit-identical to the NCCL-semantics simulation
        ref, _ = sim_nccl(m, spec, ins, peer=False)
        for g, w in zip(got, ref):
            np.testing.assert_array_equal(g, w)


def test_peer_records_replace_critical_path_all_reduces():
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.executable import Executable
    from record_sim import _dry_comms
    case = next(c for c in CASES if c["key"] == "step_tf2_bpmp_B2M2")
    m = parse_module(case["local_ir"])
    ex = Executable(m, devices=[0], comm_mode="nccl", dry=True, comm_factory=lambda e: _dry_comms(e, True))
    kinds = [k for k, _ in ex.records()]
    assert R.K_PEER in kinds
    nkeys = ex.n_peer_slots
    for k, p in ex.records():
        if k == R.K_PEER:
            assert p.n == 2 and 0 <= p.slot < nkeys and p.kind == 0
            assert p.flags[0] == ex.base + ex.flag_off * 4
            assert p.counter == ex.base + (ex.flag_off + nkeys * R.PEER_PHASES * R.PEER_MAX_BLOCKS * 8) * 4


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.session import make_nccl_comms, torch_broadcast
    text = """mesh {B:2}

func @main(%x: tensor<4x4xf32>) -> tensor<4x4xf32> {
  %r = all_reduce ["B"] %x : tensor<4x4xf32>
  %g = all_gather [["B"], []] %r : tensor<8x4xf32>
  %s = all_slice [["B"], []] %g : tensor<4x4xf32>
  %t = add %s, %r : tensor<4x4xf32>
  return %t
}
"""
    m = parse_module(text)
    seen = []

    def init(uid, n, r):
        seen.append((uid, n, r))
        return len(seen) - 1

    ex = Executable(m, devices=[rank], comm_mode="nccl", dry=True,
                    comm_factory=lambda e: make_nccl_comms(e, rank, torch_broadcast,
                                                           get_uid=lambda: os.urandom(128), init=init))
    q.put((rank, [(u.hex(), n, r) for u, n, r in seen], sorted(map(str, ex.comms))))
    dist.barrier()
    dist.destroy_process_group()


def test_comm_setup_gloo_world2():
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict((r, (seen, keys)) for r, seen, keys in (q.get(timeout=120) for _ in range(2)))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    # both ranks joined the same communicator (same uid), with NCCL ranks 0 and 1
    (s0, k0), (s1, k1) = out[0], out[1]
    assert len(s0) == len(s1) == 1
    assert s0[0][0] == s1[0][0]
    assert {s0[0][2], s1[0][2]} == {0, 1} and s0[0][1] == 2
    assert k0 == k1 == ["('B',)"]


def test_copy_engine_collectives_lowering(monkeypatch):
    """With the size threshold lifted, direct reduce-scatters become barrier +
    copy-engine pulls + a member-order fold + barrier, and gathers of function
    arguments become copy-engine pulls -- simulated across ranks, bit-identical
    to the NCCL-semantics lowering."""
    from paper_2401_11202_b200 import runtime as R
    monkeypatch.setenv("SPX_CE_MIN_BYTES", "0")
    monkeypatch.setenv("SPX_CE_RS", "1")
    seen = set()
    for key in ("rule_rs_raw", "rule_gather_merge_raw", "rule_surface_raw"):
        case = next(c for c in CASES if c["key"] == key)
        m = parse_module(case["local_ir"])
        spec = ShardingSpec.from_json(case["sharding"])
        base = parse_module(case["dense_ir"]) if "dense_ir" in case else m
        ins = case_inputs(case, base, case["seeds"][0])
        got, exs = sim_nccl(m, spec, ins, peer=True)
        for k, p in exs[0].records():
            if k == R.K_COPY:
                seen.add("copy")
            if k == R.K_PEER and p.kind == 3:
                seen.add("barrier")
        monkeypatch.setenv("SPX_CE_RS", "0")
        monkeypatch.setenv("SPX_CE_AG", "0")
        ref, _ = sim_nccl(m, spec, ins, peer=False)
        monkeypatch.setenv("SPX_CE_RS", "1")
        monkeypatch.setenv("SPX_CE_AG", "1")
        for g, w in zip(got, ref):
            np.testing.assert_array_equal(g, w)
    assert seen == {"copy", "barrier"}, seen
