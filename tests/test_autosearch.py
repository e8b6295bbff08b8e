"""AutomaticPartition search with the B200 objective.

CPU: the measured objective, fed a timer that returns the simulator's own
compute term, reproduces the reference's `plan_objective` bit for bit, so the
reference's `auto_partition` picks the same plan through it (the plumbing adds
nothing of its own).  GPU: a real measured search.  Both need the reference's
tactic front end (`spindle`): this container's /root/reference, or an install
in baseline/_ref; skipped where neither exists."""
import math
import os
import sys

import pytest

from conftest import ROOT

for _p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(_p) and _p not in sys.path:
        sys.path.append(_p)
spindle = pytest.importorskip("spindle")

from paper_2401_11202_b200.autosearch import MeasuredObjective, auto_partition_measured, b200_machine  # noqa: E402


def _sim_timer(machine):
    """All-device step time = per-device simulated compute x device count."""
    from spindle.sim import simulate

    def timer(loc, spec):
        r = simulate(loc, machine)
        return r.compute_flops / machine.peak_flops * loc.mesh.device_count
    return timer


@pytest.mark.parametrize("model,mesh,axes,budget,seed", [
    ("chain", "M:2", ["M"], 10_000, 0),          # exhaustive (test_schedule.py:231-249)
    ("mlp", "B:4,M:2", ["B", "M"], 6, 11),       # UCT sampled (test_schedule.py:263-268)
])
def test_simulated_timer_reproduces_reference_search(model, mesh, axes, budget, seed):
    from spindle.ir import Mesh
    from spindle.models import build_model
    from spindle.search import auto_partition, plan_objective
    from spindle.sim import total_flops
    m = build_model(model)
    m.mesh = Mesh.parse(mesh)
    machine = b200_machine()
    obj = MeasuredObjective(timer=_sim_timer(machine))
    plan, obj = auto_partition_measured(m, axes, budget=budget, seed=seed, machine=machine, objective=obj)
    assert plan == auto_partition(m, axes, budget=budget, seed=seed, machine=machine)
    flops = total_flops(m)
    for p, o, _, _ in obj.log:
        want = plan_objective(m, p, machine, flops)
        assert (math.isinf(o) and math.isinf(want)) or math.isclose(o, want, rel_tol=1e-12), (p, o, want)
    # identical localized programs are timed once
    assert obj.measured <= len([e for e in obj.log if math.isfinite(e[1])])
    # the reference's search module is restored afterwards
    import spindle.search as S
    assert S.plan_objective is plan_objective


@pytest.mark.gpu
def test_measured_search_on_b200():
    from spindle.ir import Mesh
    from spindle.models import build_model
    m = build_model("mlp", hidden_layers=1, batch=256, width=1024)
    m.mesh = Mesh.parse("B:2")
    plan, obj = auto_partition_measured(m, ["B"], budget=12, seed=0)
    finite = [e for e in obj.log if math.isfinite(e[1])]
    assert finite and obj.measured >= 1
    assert all(e[2] > 0 for e in finite)                 # measured per-device step time
    best = min(e[1] for e in finite)
    chosen = [e for e in finite if [s for s in e[0] if s is not None] == plan]
    assert not chosen or math.isclose(chosen[0][1], best)
