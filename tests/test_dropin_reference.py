"""The backend accepts the reference's own Module / ShardingSpec objects (the
drop-in boundary) -- checked on CPU through the record simulator
where the reference is importable (this build container), skipped elsewhere."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
if os.path.isdir(REF) and REF not in sys.path:
    sys.path.append(REF)
spindle = pytest.importorskip("spindle")

from record_sim import sim_spmd  # noqa: E402


@pytest.mark.parametrize("model,names,mesh,params", [
    ("mlp", ["bp"], "B:2", dict(hidden_layers=1, batch=16, width=8)),
    ("transformer", ["bp", "mp", "z3"], "B:2,M:2", dict(blocks=1, batch=8, d_model=8, d_ff=16)),
    ("mlp", ["bp", "es"], "B:4,M:2", {}),
])
def test_reference_objects_through_backend(model, names, mesh, params):
    from spindle.interp import interpret, random_inputs
    from spindle.ir import Mesh
    from spindle.models import build_model
    from spindle.schedule import Partitioner, cookbook_schedule
    from spindle.spmd import localize, lower_to_spmd
    from spindle.spmd_interp import relative_error, spmd_interpret as ref_spmd
    m = build_model(model, **params)
    m.mesh = Mesh.parse(mesh)
    p = Partitioner(m)
    for t in cookbook_schedule(model, names, m):
        p.apply(t)
    loc, spec = localize(lower_to_spmd(p.module))          # reference objects
    ins = random_inputs(build_model(model, **params), seed=0)
    want = ref_spmd(loc, spec, ins)
    got, _ = sim_spmd(loc, spec, ins)
    for g, w in zip(got, want):
        assert relative_error(g, w) < 1e-5


def test_divergence_error_is_the_references():
    from spindle.spmd_interp import DivergenceError as RefDiv
    from paper_2401_11202_b200 import DivergenceError
    assert issubclass(DivergenceError, RefDiv)
