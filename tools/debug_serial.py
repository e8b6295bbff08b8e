"""Run a config program's plan (a) normally (multi-stream) and (b) serially on
one stream (spx_plan_profile issues every record in order on one stream),
and compare both with the oracle: a result that is right serially but wrong
multi-stream points at a cross-stream ordering bug, wrong in both at a
kernel/layout bug."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_11202_b200 as pkg  # noqa: E402
from paper_2401_11202_b200.evaluator import _Dense, _chunk_slices, default_device  # noqa: E402
from paper_2401_11202_b200.executable import Executable  # noqa: E402
from oracle import spmd_oracle as O  # noqa: E402


def main(name, mode, scale, how):
    prog = pkg.load_program(name)
    ins = pkg.programs.synthetic_inputs(prog.dense, seed=0, scale=float(scale))
    dev = default_device()
    if mode == "spmd":
        m, want = prog.local, O.spmd_interpret(prog.local, prog.sharding, ins)
        ex = Executable(m, device=dev)
        coords = m.mesh.coords()
        per = [{n: ins[n][_chunk_slices(ins[n].shape, prog.sharding.args[n], m.mesh, c)] for n in ins} for c in coords]
    else:
        m, want = prog.dense, O.interpret(prog.dense, ins)
        ex = Executable(_Dense(m), devices=[0], device=dev)
        per = [ins]
    ex.upload_args(per)
    if how == "serial":
        ex.plan.profile()
    else:
        ex.run()
    res = ex.download_results()
    f = m.func()
    bad = []
    for j, r in enumerate(res):
        if mode == "spmd":
            from paper_2401_11202_b200.evaluator import unshard
            try:
                g = unshard(r, prog.sharding.results[j], m.mesh, coords, 1e30, "x")
            except Exception as e:
                bad.append((f.results[j], str(e)))
                continue
        else:
            g = r[0]
        e = O.relative_error(g, want[j])
        if not e < 1e-5:
            bad.append((f.results[j], float(e)))
    print(f"{name} {how}: bad {len(bad)} {bad[:6]}", flush=True)
    ex.close()


if __name__ == "__main__":
    main(*sys.argv[1:5])
