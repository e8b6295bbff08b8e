"""Measured AutomaticPartition search on one B200, printed as a table.

    python tools/autosearch_demo.py [--budget 24]

Runs the reference's auto_partition over the BP axis of the C1 MLP (mesh B:2)
and the MP axis of a 1-block transformer (mesh M:2) twice: with the
reference's simulated objective (calibrated B200 spec) and with the measured
one (autosearch.MeasuredObjective); prints each scored plan's terms.
"""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(p):
        sys.path.append(p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=int, default=24)
    args = ap.parse_args()
    from spindle.ir import Mesh
    from spindle.models import build_model
    from spindle.search import auto_partition, plan_objective
    from spindle.sim import total_flops
    from paper_2401_11202_b200.autosearch import auto_partition_measured, b200_machine
    machine = b200_machine()
    cases = [("mlp", dict(hidden_layers=1, batch=256, width=1024), "B:2", ["B"]),
             ("transformer", dict(blocks=1, batch=2048, d_model=1024, d_ff=4096), "M:2", ["M"])]
    for model, kw, mesh, axes in cases:
        m = build_model(model, **kw)
        m.mesh = Mesh.parse(mesh)
        flops = total_flops(m)
        t0 = time.time()
        sim_plan = auto_partition(m, axes, budget=args.budget, seed=0, machine=machine)
        t1 = time.time()
        plan, obj = auto_partition_measured(m, axes, budget=args.budget, seed=0, machine=machine)
        t2 = time.time()
        print(f"== {model} {kw} mesh {mesh} axes {axes} budget {args.budget}")
        print(f"simulated-objective plan ({t1 - t0:.1f} s): {sim_plan}")
        print(f"measured-objective plan  ({t2 - t1:.1f} s, {obj.measured} programs timed): {plan}")
        print(f"{'objective ms':>13} {'measured/dev ms':>15} {'comm ms':>8} {'sim ms':>8}  plan")
        seen = set()
        for p, o, t, c in sorted(obj.log, key=lambda e: e[1]):
            key = repr([s for s in p if s is not None])
            if key in seen:
                continue
            seen.add(key)
            sim = plan_objective(m, p, machine, flops)
            if math.isinf(o):
                print(f"{'inf':>13} {'-':>15} {'-':>8} {'inf':>8}  {key}")
            else:
                print(f"{o * 1e3:13.3f} {t * 1e3:15.3f} {c * 1e3:8.3f} {sim * 1e3:8.3f}  {key}")
        print()


if __name__ == "__main__":
    main()
