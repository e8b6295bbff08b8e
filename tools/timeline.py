"""Multi-stream timeline of one step (dev tool): where the main stream waits.

Runs the bench workload's program (one rank per GPU under torchrun, like
bench.py), then one traced run (runtime `spx_plan_trace`: per record the time
its stream reached it with its cross-stream waits met, and its end).  Prints,
per rank: the step span, busy time per stream, and the main-stream stalls --
gaps where the main stream sat waiting on another stream -- attributed to the
record class it waited for (the wait whose end came last).

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/timeline.py --config c3
"""
import argparse
import collections
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")


def analyse(cls, stream, ready, end, waits) -> dict:
    """Per-stream busy time and main-stream stalls of one traced run: a main
    record that became ready later than the previous main record ended waited
    for another stream -- attributed to the waited-on record whose end came
    last (its class @ its stream)."""
    ready = np.asarray(ready, dtype=np.float64)
    end = np.asarray(end, dtype=np.float64)
    n = len(cls)
    t0 = float(ready.min())
    span = float(end.max()) - t0
    busy = collections.Counter()
    by_cls = collections.Counter()
    for i in range(n):
        busy[stream[i]] += end[i] - ready[i]
        by_cls[(stream[i], cls[i])] += end[i] - ready[i]
    stalls = collections.Counter()
    stall_n = collections.Counter()
    stall_total = 0.0
    prev_end = t0
    worst = []
    for i in range(n):
        if stream[i] != 0:
            continue
        gap = ready[i] - prev_end
        if gap > 0.002 and waits[i]:
            j = max(waits[i], key=lambda w: end[w])
            key = f"{cls[j]}@s{stream[j]}"
            stalls[key] += gap
            stall_n[key] += 1
            stall_total += gap
            worst.append((gap, i, cls[i], j, cls[j], stream[j]))
        prev_end = max(prev_end, end[i])
    return {"records": n, "span_ms": round(span, 3),
            "busy_ms_by_stream": {int(k): round(v, 3) for k, v in sorted(busy.items())},
            "busy_ms_by_stream_class": {f"s{k[0]}:{k[1]}": round(v, 3) for k, v in sorted(by_cls.items())},
            "main_stall_ms": round(stall_total, 3),
            "main_stall_by_cause": {k: [round(v, 3), stall_n[k]] for k, v in stalls.most_common()},
            "worst_stalls": [{"ms": round(g, 3), "rec": i, "cls": c, "waited_on": j, "on": f"{cj}@s{sj}"}
                             for g, i, c, j, cj, sj in sorted(worst, reverse=True)[:12]]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--program", default=None)
    ap.add_argument("--json", default=None, help="write the per-record trace of rank 0 here")
    args = ap.parse_args()
    import bench
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.programs import WORKLOADS, load_program, synthetic_inputs
    from paper_2401_11202_b200.session import Session
    world, rank, local = bench.dist_env()
    dist = bench.init_dist(world, rank)
    wl = WORKLOADS[args.config]
    prog = load_program(args.program or wl["programs"][world])
    inputs = synthetic_inputs(prog.dense, seed=0, scale=wl["scale"])
    if world == 1:
        sess = Session(prog.dense, local_rank=local)
    else:
        sess = Session(prog.local, prog.sharding, mode="nccl", rank=rank, world=world, local_rank=local)
    sess.load(inputs)
    for _ in range(3):
        sess.run()
    sess.sync()
    bench.barrier(dist)
    ex = sess.ex
    ready, end = ex.plan.trace()
    bench.barrier(dist)
    ready, end = ex.plan.trace()       # second trace: warm
    names = {R.K_EW: "ew", R.K_REDUCE: "reduce", R.K_GEMM: "gemm", R.K_GATHER: "relayout",
             R.K_CREDUCE: "creduce", R.K_NCCL: "nccl", R.K_PEER: "peer", R.K_SPLIT: "split", R.K_COPY: "copy"}
    recs = ex.records()
    n = len(recs)
    stream = [0] * n
    waits = [[] for _ in range(n)]
    for idx, st, w in ex.sched:
        stream[idx] = st
        waits[idx] = list(w)
    cls = [names[k] for k, _ in recs]
    out = analyse(cls, stream, ready, end, waits)
    out["rank"] = rank
    lines = [None] * world
    if dist is not None:
        dist.all_gather_object(lines, out)
    else:
        lines = [out]
    if rank == 0:
        for o in lines:
            print(json.dumps(o), flush=True)
        if args.json:
            with open(args.json, "w") as f:
                json.dump({"cls": cls, "stream": stream, "ready": ready.tolist(), "end": end.tolist(),
                           "waits": waits}, f)
    sess.close() if hasattr(sess, "close") else None


if __name__ == "__main__":
    main()
