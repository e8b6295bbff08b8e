"""Bisect a config-program parity failure over the plan knobs (GPU)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2401_11202_b200 as pkg
from oracle import spmd_oracle as O
name, mode, scale = sys.argv[1], sys.argv[2], float(sys.argv[3])
prog = pkg.load_program(name)
ins = pkg.programs.synthetic_inputs(prog.dense, seed=0, scale=scale)
if mode == "spmd":
    want = O.spmd_interpret(prog.local, prog.sharding, ins); got = pkg.spmd_interpret(prog.local, prog.sharding, ins)
else:
    want = O.interpret(prog.dense, ins); got = pkg.interpret(prog.dense, ins)
f = (prog.local if mode == "spmd" else prog.dense).func()
errs = [(O.relative_error(g, w), f.results[j]) for j, (g, w) in enumerate(zip(got, want))]
bad = [(round(e, 9), n) for e, n in errs if not e < 1e-5]
print("worst %%.3e" %% max(e for e, _ in errs), "bad", len(bad), bad[:6])
''' % ROOT

KNOBS = [{}, {"SPX_OVERLAP": "0"}, {"SPX_GEMM_H3": "0"}, {"SPX_EW_SPLIT_FUSE": "0"}, {"SPX_SPLIT_BATCH": "0"},
         {"SPX_PDL": "0"}, {"SPX_H3_SHARE": "0"}, {"SPX_COLL_CSE": "0"}, {"SPX_EW_STATIC": "0"},
         {"SPX_SPLIT_PREFETCH": "0"}, {"SPX_CONCURRENT_GEMM": "0"}, {"SPX_UPDATE_STREAM": "0"}]

if __name__ == "__main__":
    cfgs = [a.split(":") for a in sys.argv[1:]]
    for name, mode, scale in cfgs:
        for kn in KNOBS:
            env = dict(os.environ, **kn)
            r = subprocess.run([sys.executable, "-c", CHILD, name, mode, scale], env=env, capture_output=True, text=True,
                               timeout=600)
            line = (r.stdout.strip().splitlines() or [r.stderr.strip()[-300:]])[-1]
            print(f"{name} {mode} {kn}: {line}", flush=True)
