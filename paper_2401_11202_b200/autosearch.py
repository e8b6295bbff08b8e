"""AutomaticPartition search scored on the B200.

The reference's search (`search.py:94-161`, `auto_partition`: exhaustive when
the plan space fits the budget, UCT sampling otherwise) scores every plan with
`plan_objective` (`search.py:51-73`): apply the plan to a clone, propagate,
`inf` on a PartitionError or leftover conflicts, then localize and return the
simulator's runtime (FLOPs / peak + per-collective link time and latency,
`sim.py:209-234`) plus a penalty for peak memory beyond the device's HBM.

`MeasuredObjective` keeps all of that -- the same plan application through the
reference's own rewrite / spmd passes, the same `inf` rules, the same memory
penalty and the simulator's communication term -- and replaces the FLOP term
by the measured step time of the partitioned program on a B200: the localized
module runs through this backend with every mesh device hosted on one GPU
(one batched launch per op, the evaluator's single-process mode), captured as
a CUDA graph and timed with CUDA events; that time / device count is the
per-device compute estimate.  The collective term stays the simulator's, with
the calibrated B200 spec (`machine/b200-spindle.spec`).  Identical localized
programs (different plans often localize to the same program) are measured
once.

`auto_partition_measured` runs the reference's unchanged `auto_partition` with
this objective in place of `plan_objective`, so exhaustive enumeration, UCT,
budget accounting and tie-breaking are the reference's.  The tactic front end
must be importable (`spindle`; this container's /root/reference, or an install
in baseline/_ref).
"""
from __future__ import annotations

import hashlib
import math
import os
from contextlib import contextmanager

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
B200_SPEC = os.path.join(HERE, "machine", "b200-spindle.spec")


def b200_machine():
    """The calibrated B200 MachineSpec in the reference's spec format."""
    from spindle.sim import load_machine_spec
    return load_machine_spec(B200_SPEC)


class MeasuredObjective:
    """Callable with `plan_objective`'s signature (search.py:51-52).

    timer(loc, spec) -> seconds per step for ALL mesh devices; defaults to the
    B200 measurement.  `log` keeps (plan, objective, measured_s, comm_s) per call."""

    def __init__(self, device=None, steps: int = 5, warmup: int = 2, timer=None):
        self.device = device
        self.steps = steps
        self.warmup = warmup
        self.timer = timer or self._time_on_b200
        self.cache: dict[str, float] = {}
        self.log: list[tuple] = []
        self.measured = 0

    # ---------------------------------------------------------- measurement
    def _time_on_b200(self, loc, spec) -> float:
        from .session import Session
        if self.device is None:
            from .evaluator import default_device
            self.device = default_device()
        dev = self.device
        f = loc.func()
        rng = np.random.default_rng(0)
        sess = Session(loc, spec, device=dev)
        try:
            # every mesh device's local arguments, N(0, 0.02^2) like the
            # benchmark configs (the step time does not depend on the values)
            per_device = [{n: (rng.standard_normal(tuple(t.dims)) * 0.02).astype(np.float32) for n, t in f.args}
                          for _ in loc.mesh.coords()]
            sess.ex.upload_args(per_device)
            sess.run()
            sess.sync()
            sess.capture()
            for _ in range(self.warmup):
                sess.step()
            sess.sync()
            e0, e1 = dev.event(), dev.event()
            dev.record(e0)
            for _ in range(self.steps):
                sess.step()
            dev.record(e1)
            sess.sync()
            return dev.elapsed_ms(e0, e1) / self.steps / 1e3
        finally:
            sess.close()

    # ------------------------------------------------------------ objective
    def __call__(self, module, plan, machine, model_flops, func_name: str = "main") -> float:
        from spindle.printer import print_module
        from spindle.rewrite import PartitionError, apply_atomic, apply_tile, propagate
        from spindle.search import KEEP
        from spindle.sim import simulate
        from spindle.spmd import localize, lower_to_spmd
        work = module.clone()
        f = work.func(func_name)
        try:
            for step in plan:
                if step is KEEP:
                    continue
                kind, value, dim, axis = step
                if kind == "atomic":
                    apply_atomic(f, work.mesh, value, axis, origin="auto")
                else:
                    apply_tile(f, work.mesh, value, dim, axis, origin="auto")
            conflicts = propagate(f, work.mesh, origin="auto")
        except PartitionError:
            self.log.append((list(plan), math.inf, None, None))
            return math.inf
        if conflicts:
            self.log.append((list(plan), math.inf, None, None))
            return math.inf
        loc, spec = localize(lower_to_spmd(work))
        report = simulate(loc, machine, model_flops=model_flops, func=func_name)
        comm_s = max(0.0, report.runtime_s - report.compute_flops / machine.peak_flops)
        key = hashlib.sha256((print_module(loc) + repr(sorted(spec.to_json().items()))).encode()).hexdigest()
        if key not in self.cache:
            self.cache[key] = self.timer(loc, spec)
            self.measured += 1
        ndev = loc.mesh.device_count if loc.mesh is not None else 1
        t_dev = self.cache[key] / ndev
        over = max(0.0, report.peak_memory_bytes - machine.hbm_bytes)
        obj = t_dev + comm_s + over / machine.link_bandwidth
        self.log.append((list(plan), obj, t_dev, comm_s))
        return obj


@contextmanager
def objective_in_place(objective):
    """Swap the reference search's `plan_objective` for `objective`."""
    from spindle import search
    saved = search.plan_objective
    search.plan_objective = objective
    try:
        yield
    finally:
        search.plan_objective = saved


def auto_partition_measured(module, axes: list[str], budget: int = 64, seed: int = 0, machine=None,
                            func_name: str = "main", objective: MeasuredObjective | None = None):
    """The reference's `auto_partition` (search.py:94-161) with the B200 as the
    objective.  Returns (plan, objective) -- the objective's `log` holds every
    scored plan."""
    from spindle import search
    objective = objective or MeasuredObjective()
    machine = machine or b200_machine()
    with objective_in_place(objective):
        plan = search.auto_partition(module, axes, budget=budget, seed=seed, machine=machine,
                                     func_name=func_name)
    return plan, objective
