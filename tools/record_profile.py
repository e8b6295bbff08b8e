"""Per-record timing of one benchmark step (eager, events between records):
kind, shape, time, algorithmic bytes / flops and the achieved rate.  Dev tool.

    python tools/record_profile.py [--program c2_tf8_dense] [--top 30]
"""
import argparse
import collections
import sys

import numpy as np

sys.path.insert(0, ".")


def ew_bytes(p):
    """Distinct bytes an EW record touches: each input view's extent + outputs."""
    dims = [int(p.dims[j]) for j in range(p.rank)]
    total = 0
    for i in range(p.n_in):
        v = p.inp[i]
        ext = 1
        for j in range(p.rank):
            if int(v.stride[j]) != 0:
                ext *= dims[j]
        total += ext * 4
    return total + p.n_out * int(np.prod(dims)) * 4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--program", default="c2_tf8_dense")
    ap.add_argument("--top", type=int, default=30)
    args = ap.parse_args()
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.programs import load_program, synthetic_inputs
    from paper_2401_11202_b200.session import Session
    p = load_program(args.program)
    sess = Session(p.dense if p.local is None else p.local, p.sharding)
    sess.load(synthetic_inputs(p.dense, seed=0, scale=0.02))
    sess.run()
    sess.sync()
    ms = sess.ex.plan.profile()
    ms = sess.ex.plan.profile()
    rows = []
    cls = collections.Counter()
    for (kind, prm), t in zip(sess.ex.records(), ms):
        if kind == R.K_GEMM:
            fl = 2.0 * prm.M * prm.N * prm.K * prm.ndev
            desc = f"gemm {prm.M}x{prm.N}x{prm.K} amn={prm.a_mn_major} bk={prm.b_k_major} splits={prm.splits}"
            rate = f"{3 * fl / (t * 1e-3) / 1e12:7.1f} TF/s(tf32)"
            name = "gemm"
        elif kind == R.K_EW:
            b = ew_bytes(prm)
            dims = [int(prm.dims[j]) for j in range(prm.rank)]
            desc = f"ew dims={dims} in={prm.n_in} out={prm.n_out} prog={prm.n_prog} vec={prm.vec}"
            rate = f"{b / (t * 1e-3) / 1e9:7.0f} GB/s"
            name = "ew"
        elif kind == R.K_REDUCE:
            b = ew_bytes(prm.x)
            desc = (f"reduce mode={prm.mode} kept={[int(prm.kept_dims[j]) for j in range(prm.n_kept)]} "
                    f"red={[int(prm.red_dims[j]) for j in range(prm.n_red)]}")
            rate = f"{b / (t * 1e-3) / 1e9:7.0f} GB/s"
            name = "reduce"
        else:
            desc, rate, name = f"kind {kind}", "", f"k{kind}"
        cls[name] += t
        rows.append((t, desc, rate))
    tot = sum(ms)
    print(f"total {tot:.3f} ms over {len(ms)} records; by class: "
          + ", ".join(f"{k} {v:.3f}" for k, v in cls.most_common()))
    agg = collections.defaultdict(lambda: [0, 0.0, ""])
    for t, d, r in rows:
        a = agg[d]
        a[0] += 1
        a[1] += t
        a[2] = r
    for d, (n, t, r) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:args.top]:
        print(f"{t:8.3f} ms {100 * t / tot:5.1f}% x{n:3d}  {r:>18s}  {d}")


if __name__ == "__main__":
    main()
