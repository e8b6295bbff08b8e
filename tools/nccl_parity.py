"""Multi-GPU parity (one process per GPU, NCCL collectives).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nccl_parity.py

Runs every golden case whose mesh has N devices through Session(mode="nccl"),
reassembles the results on rank 0 (unshard + replica consensus) and compares
them with the reference's golden outputs (tests/golden).  Exit 1 on failure.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch.distributed as dist
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import case_expected, case_inputs, golden_cases
    from paper_2401_11202_b200 import parse_module, ShardingSpec
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.evaluator import relative_error, unshard, DivergenceError
    from paper_2401_11202_b200.session import Session
    import torch
    ngpu = max(1, torch.cuda.device_count())
    dev = R.Device(local % ngpu)      # 8 ranks on a 4-GPU box: two processes per GPU (SPX_NCCL_NONE=1)
    fails, n = [], 0
    for case in golden_cases():
        if "local_ir" not in case:
            continue
        m = parse_module(case["local_ir"])
        if m.mesh.device_count != world:
            continue
        spec = ShardingSpec.from_json(case["sharding"])
        base = parse_module(case["dense_ir"]) if "dense_ir" in case else m
        for s in case["seeds"][:1]:
            ins = case_inputs(case, base, s)
            try:
                sess = Session(m, spec, mode="nccl", device=dev, rank=rank, world=world, local_rank=local)
            except Exception:           # SPX_NCCL_NONE=1 and a collective that needs NCCL
                continue
            sess.load(ins)
            sess.run()
            sess.sync()
            # graph replay must reproduce the eager run
            sess.capture()
            sess.step()
            sess.sync()
            res = [r[0] for r in sess.results()]
            sess.close()
            allres = [None] * world
            dist.all_gather_object(allres, res)
            if rank == 0:
                n += 1
                coords = m.mesh.coords()
                try:
                    got = [unshard([allres[r][j] for r in range(world)], spec.results[j], m.mesh, coords,
                                   1e-5, f"result {j}") for j in range(len(res))]
                    if case.get("error") == "DivergenceError":
                        fails.append((case["key"], "expected DivergenceError"))
                        continue
                    worst = max(relative_error(g, w) for g, w in zip(got, case_expected(case, s, "spmd")))
                    if not worst < 1e-5 or not all(np.all(np.isfinite(g)) for g in got):
                        fails.append((case["key"], worst))
                except DivergenceError as e:
                    if case.get("error") != "DivergenceError":
                        fails.append((case["key"], str(e)))
    # the BASELINE configs' own programs at this world size, default knobs:
    # eager run and graph replay vs the oracle, executed collectives vs the
    # simulator's counts (runtime counters)
    from oracle import spmd_oracle as O
    from paper_2401_11202_b200.programs import load_program, synthetic_inputs
    cfg = {2: [("c1_mlp_bp_B2", 0.25), ("c2_tf8_bp_B2", 0.02), ("c3_tf1_bpz3_B2", 0.02), ("c4_unet_bpz2_B2", 0.05),
               ("c5_tf8_bpz3_B2", 0.02)],
           4: [("c2_tf8_bpmp_B2M2", 0.02), ("c3_tf1_bpz3_B4", 0.02), ("c4_unet_bpz2_B4", 0.05),
               ("c5_tf8_bpmpz3_B2M2", 0.02)],
           8: [("c2_tf1_bpmp_B2M4", 0.02), ("c3_tf1_bpz3_B8", 0.02), ("c4_unet_bpz2_B8", 0.05),
               ("c5_tf1_bpmpz3emb_B2M2E2", 0.02)]}.get(world, [])
    only = os.environ.get("PARITY_CONFIGS")
    for name, scale in cfg:
        if only and name not in only.split(","):
            continue
        prog = load_program(name)
        m, spec = prog.local, prog.sharding
        ins = synthetic_inputs(prog.dense, seed=0, scale=scale)
        try:
            sess = Session(m, spec, mode="nccl", device=dev, rank=rank, world=world, local_rank=local)
        except Exception as e:          # SPX_NCCL_NONE=1 and a collective that needs NCCL
            if rank == 0:
                print(f"{name}: skipped ({str(e)[:120]})", flush=True)
            continue
        sess.load(ins)
        sess.run()
        sess.sync()
        eager = [r[0] for r in sess.results()]
        sess.capture()
        sess.step()
        sess.sync()
        replay = [r[0] for r in sess.results()]
        work = sess.ex.work_report()
        pred = sess.ex.issued_per_run()["coll"]
        sess.close()
        same = all(np.array_equal(a, b) for a, b in zip(eager, replay))
        allres = [None] * world
        dist.all_gather_object(allres, (replay, same, work["collectives"]["executed"] == pred))
        if rank == 0:
            n += 1
            coords = m.mesh.coords()
            want = O.spmd_interpret(m, spec, ins)
            try:
                got = [unshard([allres[r][0][j] for r in range(world)], spec.results[j], m.mesh, coords,
                               1e-5, f"result {j}") for j in range(len(want))]
                worst = max(relative_error(g, w) for g, w in zip(got, want))
                fin = all(np.all(np.isfinite(g)) for g in got)
                print(f"{name}: worst rel err {worst:.3e} finite {fin} replay==eager "
                      f"{all(a[1] for a in allres)} counters==records {all(a[2] for a in allres)} "
                      f"executed {work['collectives']['executed']} program {work['collectives']['program']}",
                      flush=True)
                if not worst < 1e-5 or not fin or not all(a[1] and a[2] for a in allres):
                    fails.append((name, worst))
            except DivergenceError as e:
                fails.append((name, str(e)))
    # large all_reduce over every rank (the peer-memory kernels: one-shot for 2
    # members, two-shot for 4 / 8): bit-identical to the member-order fold
    for rows in (1024, 257):
        text = (f"mesh {{M:{world}}}\n\nfunc @main(%x: tensor<{rows}x1024xf32>) -> tensor<{rows}x1024xf32> {{\n"
                f"  %r = all_reduce [\"M\"] %x : tensor<{rows}x1024xf32>\n  return %r\n}}\n")
        m = parse_module(text)
        spec = ShardingSpec({"x": [[], []]}, [[[], []]])
        xs = [np.random.default_rng(100 + r).standard_normal((rows, 1024)).astype(np.float32) for r in range(world)]
        sess = Session(m, spec, mode="nccl", device=dev, rank=rank, world=world, local_rank=local)
        sess.ex.upload_args([{"x": xs[rank]}])
        sess.run()
        sess.sync()
        got = sess.results()[0][0]
        kinds = sorted({k for k, _ in sess.ex.records()})
        sess.close()
        want = xs[0].copy()
        for x in xs[1:]:
            want = want + x
        allok = [None] * world
        dist.all_gather_object(allok, bool(np.array_equal(got, want)))
        if rank == 0:
            n += 1
            if not all(allok):
                fails.append((f"all_reduce_{rows}x1024", "not bit-identical to the member-order fold"))
            if world > 1 and R.K_PEER not in kinds:
                fails.append((f"all_reduce_{rows}x1024", "peer kernel not used"))
    if rank == 0:
        print(json.dumps({"world": world, "cases": n, "failures": fails}))
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and fails:
        sys.exit(1)


if __name__ == "__main__":
    main()
