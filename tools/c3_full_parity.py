"""C3 at its full size (32 blocks, d_model 2048, d_ff 8192, batch 8192) --
the N=1 benchmark program -- through the drop-in `interpret` on the GPU vs
the oracle restatement of the reference evaluator on the host (~90 GB of
host RAM, ~1-2 min per step), as a training loop of STEPS steps with the
updated parameters and momenta fed back.  Prints per step the loss of both
and the worst relative error over all outputs."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_11202_b200 as pkg  # noqa: E402
from paper_2401_11202_b200.programs import load_program, synthetic_inputs  # noqa: E402
from oracle import spmd_oracle as O  # noqa: E402


def feed(f, cur, out):
    for j, r in enumerate(f.results):
        if r.startswith("new_") and r[4:] in cur:
            cur[r[4:]] = out[j]


def main():
    name = os.environ.get("PROGRAM", "c3_tf32_dense")
    steps = int(os.environ.get("STEPS", "2"))
    p = load_program(name)
    m, f = p.dense, p.dense.func()
    a = synthetic_inputs(m, 0, 0.02)
    b = dict(a)
    for it in range(steps):
        t0 = time.perf_counter()
        og = pkg.interpret(m, a)
        t1 = time.perf_counter()
        oo = O.interpret(m, b)
        t2 = time.perf_counter()
        errs = [O.relative_error(x, y) for x, y in zip(og, oo)]
        fin_g = all(np.isfinite(x).all() for x in og)
        fin_o = all(np.isfinite(x).all() for x in oo)
        worst = max(errs) if fin_g and fin_o else float("nan")
        print(f"{name} step {it}: loss gpu {float(og[0]):.6f} oracle {float(oo[0]):.6f}; finite gpu {fin_g} "
              f"oracle {fin_o}; worst rel err over {len(errs)} outputs {worst:.3e}; gpu call {t1 - t0:.2f} s, "
              f"oracle {t2 - t1:.1f} s", flush=True)
        feed(f, a, og)
        feed(f, b, oo)
        del og, oo


if __name__ == "__main__":
    main()
