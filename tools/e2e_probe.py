"""Drop-in call as a training loop (results new_X fed back as arguments X):
(1) C2 dense on the GPU vs the oracle, step by step; (2) C3 dense on the GPU,
loss per step and the time of each phase of the call (copy in, step, copy out)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_11202_b200 as pkg  # noqa: E402
from paper_2401_11202_b200 import evaluator as E  # noqa: E402
from paper_2401_11202_b200 import runtime as R  # noqa: E402
from paper_2401_11202_b200.programs import load_program, synthetic_inputs  # noqa: E402
from oracle import spmd_oracle as O  # noqa: E402


def feed(f, cur, out):
    for j, r in enumerate(f.results):
        if r.startswith("new_") and r[4:] in cur:
            cur[r[4:]] = out[j]


def parity(name, steps):
    p = load_program(name)
    m, f = p.dense, p.dense.func()
    a = synthetic_inputs(m, 0, 0.02)
    b = dict(a)
    for it in range(steps):
        og = pkg.interpret(m, a)
        oo = O.interpret(m, b)
        err = max(O.relative_error(x, y) for x, y in zip(og, oo))
        print(f"{name} step {it}: loss gpu {float(og[0]):.6f} oracle {float(oo[0]):.6f} worst rel err {err:.2e} "
              f"finite {all(np.isfinite(x).all() for x in og)}", flush=True)
        feed(f, a, og)
        feed(f, b, oo)


def phases(name, steps):
    """C3 through the drop-in call with its copies in the plan (io mode), the
    same pinned arguments every call (no feedback: the model diverges)."""
    p = load_program(name)
    m = p.dense
    pool = R.pinned_pool()
    cur = {}
    for k, v in synthetic_inputs(m, 0, 0.02).items():
        x = pool.array(v.shape, v.dtype)
        x[...] = v
        cur[k] = x
    for it in range(steps):
        t0 = time.perf_counter()
        out = pkg.interpret(m, cur)
        t1 = time.perf_counter()
        print(f"{name} call {it}: {t1 - t0:.3f}s loss {float(out[0]):.4f} finite "
              f"{all(np.isfinite(x).all() for x in out)} pool {pool.total / 1e9:.1f} GB", flush=True)
        del out
    os.environ["SPX_IO_OVERLAP"] = "0"
    for it in range(3):
        t0 = time.perf_counter()
        out = pkg.interpret(m, cur)
        print(f"{name} SPX_IO_OVERLAP=0 call {it}: {time.perf_counter() - t0:.3f}s loss {float(out[0]):.4f}", flush=True)
        del out


if __name__ == "__main__":
    if os.environ.get("PARITY", "1") != "0":
        parity("c2_tf8_dense", int(os.environ.get("STEPS", "8")))
    phases("c3_tf32_dense", int(os.environ.get("STEPS", "8")))
