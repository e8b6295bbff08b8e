"""Program cache generator (test/bench infrastructure; runs only where the
reference is importable, i.e. in the build container, never on the GPU box).

Partitions each benchmark configuration with the reference's UNCHANGED tactic
API (`Partitioner` + `cookbook_schedule`, /root/reference/pkg/src/spindle/
schedule.py:194-295, :309-338), lowers and localizes it
(`localize(lower_to_spmd(...))`, spmd.py:212-261) and writes the artefacts the
reference's own CLI dumps (`cli.py:79-91`):

    programs/<name>/dense.ir       the unpartitioned module (interpret semantics)
    programs/<name>/local.ir       the localized per-device SPMD module
    programs/<name>/sharding.json  ShardingSpec.to_json()
    programs/<name>/meta.json      counts (collective_counts), simulator cost
                                   (simulate(...).to_json()), model params,
                                   schedule, mesh, partition wall time

This is the "cached artefact format" of SURVEY.md §8(f) rank 2: partitioning
deep models takes minutes to hours, evaluating them does not.

Partitioning runs under `fast_partitioning()` (paper_2401_11202_b200/fastpart.py:
indexed find_def/collect_uses, identical output); --slow uses the reference as is.

usage: PYTHONPATH=/root/reference/pkg/src python tools/make_programs.py [--slow] NAME [NAME...]
       PYTHONPATH=/root/reference/pkg/src python tools/make_programs.py --list
"""
from __future__ import annotations

import contextlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_11202_b200.fastpart import fast_partitioning  # noqa: E402

SLOW = False

OUT = os.environ.get("SPX_PROGRAMS_OUT") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2401_11202_b200", "programs")

TF_C2 = dict(blocks=8, batch=2048, d_model=1024, d_ff=4096)
TF_C3 = dict(blocks=32, batch=8192, d_model=2048, d_ff=8192)
MLP_C1 = dict(hidden_layers=1, batch=256, width=1024)

# name -> (model, params, mesh or None (dense only), cookbook stages, extra tactics)
EMB = ("E", {"x": 1, "y": 1})   # EMB-analog: shard activations along d_model
UNET_C4 = dict(batch=128, height=32, width=32, c0=64, c1=256, c2=512)

CONFIGS = {
    # C1: 2-layer MLP (1 hidden layer = 2 linear layers) b=256 d=1024, BP on B:2
    "c1_mlp_bp_B2": ("mlp", MLP_C1, "B:2", ["bp"], []),
    "c1_mlp_dense": ("mlp", MLP_C1, None, [], []),
    # C2: transformer 8 blocks d=1024, BP+MP on 2x4; scaling meshes 2x2, 2
    "c2_tf8_dense": ("transformer", TF_C2, None, [], []),
    "c2_tf8_bp_B2": ("transformer", TF_C2, "B:2", ["bp"], []),
    "c2_tf8_bpmp_B2M2": ("transformer", TF_C2, "B:2,M:2", ["bp", "mp"], []),
    "c2_tf8_bp_B4": ("transformer", TF_C2, "B:4", ["bp"], []),
    "c2_tf8_bpmp_B2M4": ("transformer", TF_C2, "B:2,M:4", ["bp", "mp"], []),
    # C3: transformer 32 blocks d=2048, BP+Z3 on B:8 (+ B:4, B:2)
    "c3_tf32_dense": ("transformer", TF_C3, None, [], []),
    "c3_tf32_bpz3_B8": ("transformer", TF_C3, "B:8", ["bp", "z3"], []),
    "c3_tf32_bpz3_B4": ("transformer", TF_C3, "B:4", ["bp", "z3"], []),
    "c3_tf32_bpz3_B2": ("transformer", TF_C3, "B:2", ["bp", "z3"], []),
    # C4: U-Net analog (tools/unet_model.py), BP+Z2 on B:8 (+ B:4, B:2)
    "c4_unet_dense": ("unet", UNET_C4, None, [], []),
    "c4_unet_bpz2_B8": ("unet", UNET_C4, "B:8", ["bp", "z2"], []),
    "c4_unet_bpz2_B4": ("unet", UNET_C4, "B:4", ["bp", "z2"], []),
    "c4_unet_bpz2_B2": ("unet", UNET_C4, "B:2", ["bp", "z2"], []),
    # C5: transformer 8 blocks d=1024, BP+MP+Z3+EMB on 2x2x2 (+ 2x2, 2)
    "c5_tf8_bpmpz3emb_B2M2E2": ("transformer", TF_C2, "B:2,M:2,E:2", ["bp", "mp", "z3"], [EMB]),
    "c5_tf8_bpmpz3_B2M2": ("transformer", TF_C2, "B:2,M:2", ["bp", "mp", "z3"], []),
    "c5_tf8_bpz3_B2": ("transformer", TF_C2, "B:2", ["bp", "z3"], []),
    # parity programs: the BASELINE configs' own meshes and tactics at full
    # width and reduced depth (blocks are identical; the CPU oracle cannot hold
    # C3 at 32 blocks) -- tests/test_config_parity.py
    "c2_tf1_bpmp_B2M4": ("transformer", dict(TF_C2, blocks=1), "B:2,M:4", ["bp", "mp"], []),
    "c2_tf2_bpmp_B2M4": ("transformer", dict(TF_C2, blocks=2), "B:2,M:4", ["bp", "mp"], []),
    "c5_tf1_bpmpz3emb_B2M2E2": ("transformer", dict(TF_C2, blocks=1), "B:2,M:2,E:2", ["bp", "mp", "z3"], [EMB]),
    "c5_tf2_bpmpz3emb_B2M2E2": ("transformer", dict(TF_C2, blocks=2), "B:2,M:2,E:2", ["bp", "mp", "z3"], [EMB]),
    "c3_tf1_bpz3_B8": ("transformer", dict(TF_C3, blocks=1), "B:8", ["bp", "z3"], []),
    # CPU-baseline sample for C3 (t(1) + 31 (t(2) - t(1)))
    "c3_tf1_dense": ("transformer", dict(TF_C3, blocks=1), None, [], []),
    "c3_tf2_dense": ("transformer", dict(TF_C3, blocks=2), None, [], []),
}
# ... and for the reference arm at N > 1 (the partitioned program's CPU evaluator)
for _n in (2, 4, 8):
    for _b in (1, 2):
        CONFIGS[f"c3_tf{_b}_bpz3_B{_n}"] = ("transformer", dict(TF_C3, blocks=_b), f"B:{_n}", ["bp", "z3"], [])


def make(name: str):
    from spindle.ir import Mesh
    from spindle.models import build_model
    from spindle.printer import print_module
    from spindle.schedule import ManualPartition, Partitioner, cookbook_schedule

    model, params, mesh, stages, extra = CONFIGS[name]
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    if model == "unet":
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from unet_model import unet_schedule, unet_train
        build = lambda: unet_train(**params)
        schedule = lambda names, m: unet_schedule(names, m)
    else:
        build = lambda: build_model(model, **params)
        schedule = lambda names, m: cookbook_schedule(model, names, m)
    module = build()
    meta = {"name": name, "model": model, "params": params, "mesh": mesh,
            "schedule": stages + [f"manual@{ax}:{json.dumps(s)}" for ax, s in extra]}
    with open(os.path.join(d, "dense.ir"), "w") as fh:
        fh.write(print_module(module))
    if mesh is not None:
        module.mesh = Mesh.parse(mesh)
        t0 = time.perf_counter()
        p = Partitioner(module)
        ctx = contextlib.nullcontext() if SLOW else fast_partitioning()
        with ctx:
            for t in schedule(stages, module):
                p.apply(t)
            for ax, s in extra:
                p.apply(ManualPartition(ax, dict(s)))
        ex = p.export()
        meta["partition_s"] = time.perf_counter() - t0
        meta["partitioner"] = "reference" if SLOW else "reference + fastpart index"
        meta["counts"] = ex["counts"]
        meta["cost"] = ex["cost"]
        meta["conflicts"] = sum(len(r["conflicts"]) for r in ex["reports"])
        with open(os.path.join(d, "local.ir"), "w") as fh:
            fh.write(ex["local_ir"])
        with open(os.path.join(d, "sharding.json"), "w") as fh:
            json.dump(ex["sharding"], fh)
    from spindle.sim import total_flops
    meta["model_flops"] = total_flops(build())
    with open(os.path.join(d, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{name}: done {meta.get('partition_s', 0):.1f}s counts={meta.get('counts')}",
          flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["--list"]:
        print("\n".join(CONFIGS))
        sys.exit(0)
    names = sys.argv[1:]
    if "--slow" in names:
        SLOW = True
        names.remove("--slow")
    for n in names:
        make(n)
