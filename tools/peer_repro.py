"""Repro harness for multi-GPU peer-collective issues (dev tool).

    torchrun --nproc-per-node N tools/peer_repro.py PROGRAM MODE STEPS
MODE: eager (plan.run per step, sync each step) | graph (replay, sync at end)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch.distributed as dist
    prog_name, mode, steps = sys.argv[1], sys.argv[2], int(sys.argv[3])
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_11202_b200.programs import load_program, synthetic_inputs
    from paper_2401_11202_b200.session import Session
    p = load_program(prog_name)
    sess = Session(p.local, p.sharding, mode="nccl", rank=rank, world=world, local_rank=rank)
    sess.load(synthetic_inputs(p.dense, seed=0, scale=0.05))
    if mode == "graph":
        sess.capture()
    t0 = time.time()
    for i in range(steps):
        if mode == "eager":
            sess.run()
            sess.sync()
        else:
            sess.step()
    sess.sync()
    dist.barrier()
    if rank == 0:
        print(f"{prog_name} {mode} {steps} steps ok in {time.time() - t0:.2f}s", flush=True)


if __name__ == "__main__":
    main()
