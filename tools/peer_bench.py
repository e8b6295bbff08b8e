"""Chained all-reduce latency, one process per GPU (dev tool).

    torchrun --nproc-per-node N tools/peer_bench.py [--mb 4] [--chain 32]

Times a CUDA-graph replay of CHAIN dependent all_reduce ops over all N ranks
(the activation all-reduces of Megatron-style model parallelism) through
Session(mode="nccl"); SPX_PEER=0 selects NCCL, 1 the peer-memory kernel.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=float, default=4.0)
    ap.add_argument("--chain", type=int, default=32)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch.distributed as dist
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.ir import ShardingSpec, parse_module
    from paper_2401_11202_b200.session import Session
    cols = 1024
    rows = max(1, int(args.mb * (1 << 20) / 4 / cols))
    t = f"tensor<{rows}x{cols}xf32>"
    lines = [f"mesh {{M:{world}}}", "", f"func @main(%x: {t}) -> {t} {{"]
    prev = "%x"
    for i in range(args.chain):
        lines.append(f'  %a{i} = all_reduce ["M"] {prev} : {t}')
        prev = f"%a{i}"
    lines += [f"  return {prev}", "}", ""]
    m = parse_module("\n".join(lines))
    spec = ShardingSpec({"x": [[], []]}, [[[], []]])
    dev = R.Device(local)
    sess = Session(m, spec, mode="nccl", device=dev, rank=rank, world=world, local_rank=local)
    x = np.full((rows, cols), 1.0 / world, dtype=np.float32)
    sess.load({"x": x})
    sess.run()
    sess.sync()
    sess.capture()
    for _ in range(3):
        sess.step()
    sess.sync()
    e0, e1 = dev.event(), dev.event()
    dist.barrier()
    dev.record(e0)
    for _ in range(args.iters):
        sess.step()
    dev.record(e1)
    dev.sync()
    ms = dev.elapsed_ms(e0, e1) / args.iters
    kinds = sorted({k for k, _ in sess.ex.records()})
    if rank == 0:
        print(json.dumps({"world": world, "mb": rows * cols * 4 / 2**20, "chain": args.chain,
                          "us_per_allreduce": ms * 1e3 / args.chain, "peer": R.K_PEER in kinds}))
    sess.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
