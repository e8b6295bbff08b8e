"""§8(f) rank 1: the indexed partitioner lookups (fastpart.py) give the
reference partitioner's exact output -- every lookup cross-checked against the
reference's own walk (verify mode), and the exported localized IR, sharding
and collective counts compared with an unpatched run."""
import json
import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")


def _partition(model, params, mesh, stages, fast, verify=False):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from spindle.ir import Mesh
    from spindle.models import build_model
    from spindle.schedule import Partitioner, cookbook_schedule
    from paper_2401_11202_b200.fastpart import fast_partitioning
    m = build_model(model, **params)
    m.mesh = Mesh.parse(mesh)
    p = Partitioner(m)
    if fast:
        with fast_partitioning(verify=verify) as st:
            for t in cookbook_schedule(model, stages, m):
                p.apply(t)
        assert st.hits > 0
    else:
        for t in cookbook_schedule(model, stages, m):
            p.apply(t)
    return p.export()


@pytest.mark.parametrize("model,params,mesh,stages", [
    ("mlp", dict(hidden_layers=2, batch=64, width=64), "B:2", ["bp"]),
    ("mlp", dict(hidden_layers=2, batch=64, width=64), "B:2,M:2", ["bp", "mp", "z3"]),
    ("transformer", dict(blocks=1, batch=64, d_model=32, d_ff=64), "B:2,M:2", ["bp", "mp"]),
    ("transformer", dict(blocks=2, batch=64, d_model=32, d_ff=64), "B:2,M:2", ["bp", "mp", "z3"]),
    ("transformer", dict(blocks=1, batch=64, d_model=32, d_ff=64), "B:4", ["bp", "z2"]),
])
def test_fast_partitioning_identical(model, params, mesh, stages):
    slow = _partition(model, params, mesh, stages, fast=False)
    fast = _partition(model, params, mesh, stages, fast=True, verify=True)
    assert fast["local_ir"] == slow["local_ir"]
    assert json.dumps(fast["sharding"], sort_keys=True) == json.dumps(slow["sharding"], sort_keys=True)
    assert fast["counts"] == slow["counts"]


def test_patch_is_scoped():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from spindle import ir, rewrite
    from paper_2401_11202_b200.fastpart import fast_partitioning
    before = (ir.find_def, ir.collect_uses, rewrite.find_def, rewrite.apply_tile)
    with fast_partitioning():
        assert ir.find_def is not before[0] and rewrite.apply_tile is not before[3]
    assert (ir.find_def, ir.collect_uses, rewrite.find_def, rewrite.apply_tile) == before
