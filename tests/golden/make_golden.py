"""Golden-vector generator: runs the REFERENCE itself (importable only in the
build container: PYTHONPATH=/root/reference/pkg/src) and records its outputs
so the oracle restatement (oracle/spmd_oracle.py) and the CUDA backend can be
pinned to them on machines where the reference does not exist.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/cases.json (programs as canonical IR text, sharding specs,
input recipes, expected errors) and tests/golden/outputs.npz (reference
outputs).  Sources of the cases (all in /root/reference/pkg/tests):
  * hand-written collective programs of test_spmd.py:56-171, :292-334 and
    test_parser.py:72-95 (fused with the reference's fuse_collectives, so
    reduce_scatter / all_to_all / multi-axis layouts appear), run through
    spmd_interpret with replicated inputs like `same_behavior` (:38-53);
  * the acceptance matrix of test_acceptance.py:64-92 (every model x cookbook
    schedule on B:4,M:2 / M:2) at the reference's toy sizes, partitioned with
    the unchanged tactic API, run through interpret and spmd_interpret;
  * small training steps at the benchmark configs' structure (mlp BP on B:2,
    transformer BP+MP / BP+Z3 / BP+MP+Z3+EMB) -- SURVEY.md §8(d);
  * one-op dense programs in the style of conftest.direct_op_module
    (conftest.py:24-31) and test_acceptance._op_sites (:284-310).
"""
from __future__ import annotations

import json
import os

import numpy as np

from spindle.interp import interpret, random_inputs
from spindle.ir import FuncBuilder, Mesh, TensorType
from spindle.models import build_model
from spindle.parser import parse_module
from spindle.printer import print_module
from spindle.schedule import ManualPartition, Partitioner, cookbook_schedule
from spindle.spmd import ShardingSpec, collective_counts, fuse_collectives, localize, lower_to_spmd
from spindle.spmd_interp import DivergenceError, spmd_interpret
from spindle.sim import BUILTIN_SPECS, simulate

HERE = os.path.dirname(os.path.abspath(__file__))

RULE_PROGRAMS = {
    "rs": ("""mesh {K:2}

func @main(%x: tensor<4x4xf32>) -> tensor<2x4xf32> {
  %r = all_reduce ["K"] %x : tensor<4x4xf32>
  %s = all_slice [["K"], []] %r : tensor<2x4xf32>
  return %s
}
""", [[["K"], []]]),
    "a2a": ("""mesh {K:2}

func @main(%x: tensor<2x4xf32>) -> tensor<4x2xf32> {
  %g = all_gather [["K"], []] %x : tensor<4x4xf32>
  %s = all_slice [[], ["K"]] %g : tensor<4x2xf32>
  return %s
}
""", [[[], ["K"]]]),
    "cancel": ("""mesh {K:2}

func @main(%x: tensor<2x4xf32>) -> tensor<2x4xf32> {
  %g = all_gather [["K"], []] %x : tensor<4x4xf32>
  %s = all_slice [["K"], []] %g : tensor<2x4xf32>
  return %s
}
""", None),
    "commute": ("""mesh {A:2, B:2}

func @main(%x: tensor<4x4xf32>) -> tensor<2x4xf32> {
  %r = all_reduce ["A"] %x : tensor<4x4xf32>
  %s = all_slice [["B"], []] %r : tensor<2x4xf32>
  return %s
}
""", [[["B"], []]]),
    "max_rs": ("""mesh {K:2}

func @main(%x: tensor<4x4xf32>) -> tensor<2x4xf32> {
  %r = all_reduce<max> ["K"] %x : tensor<4x4xf32>
  %s = all_slice [["K"], []] %r : tensor<2x4xf32>
  return %s
}
""", [[["K"], []]]),
    "slice_merge": ("""mesh {A:2, B:2}

func @main(%x: tensor<4x4xf32>) -> tensor<2x2xf32> {
  %a = all_slice [["A"], []] %x : tensor<2x4xf32>
  %b = all_slice [[], ["B"]] %a : tensor<2x2xf32>
  return %b
}
""", [[["A"], ["B"]]]),
    "gather_merge": ("""mesh {A:2, B:2}

func @main(%x: tensor<2x2xf32>) -> tensor<4x4xf32> {
  %a = all_gather [[], ["B"]] %x : tensor<2x4xf32>
  %b = all_gather [["A"], []] %a : tensor<4x4xf32>
  return %b
}
""", None),
    "surface": ("""mesh {B:4, M:2}

func @main(%x: tensor<8x8xf32>) -> tensor<8x8xf32> {
  %g = all_gather [["B"], []] %x : tensor<32x8xf32>
  %r = all_reduce ["M"] %g : tensor<32x8xf32>
  %s = all_slice [["B"], ["M"]] %r : tensor<8x4xf32>
  %t = all_to_all 0->1 ["M"] %s : tensor<16x2xf32>
  %c = reduce_scatter ["M"] [["M"], []] %t : tensor<8x2xf32>
  %o = all_gather [[], ["M"]] %c : tensor<8x4xf32>
  %p = all_gather [[], ["M"]] %o : tensor<8x8xf32>
  return %p
}
""", None),
    "multiaxis": ("""mesh {A:2, B:2, C:2}

func @main(%x: tensor<8x8xf32>, %y: tensor<8x8xf32>) -> (tensor<8x8xf32>, tensor<2x4xf32>, tensor<8x16xf32>) {
  %s = all_slice [["C", "A"], ["B"]] %x : tensor<2x4xf32>
  %e = exp %s : tensor<2x4xf32>
  %g = all_gather [["C", "A"], ["B"]] %e : tensor<8x8xf32>
  %r = all_reduce ["B", "A"] %s : tensor<2x4xf32>
  %m = all_reduce<max> ["C"] %r : tensor<2x4xf32>
  %t = all_slice [[], ["A", "C"]] %y : tensor<8x2xf32>
  %a = all_to_all 1->0 ["B"] %t : tensor<4x4xf32>
  %q = all_gather [["B"], []] %a : tensor<8x4xf32>
  %u = all_gather [[], ["A", "C"]] %q : tensor<8x16xf32>
  return %g, %m, %u
}
""", [[[], []], [["C", "A"], ["B"]], [[], []]]),
    "ones_ar": ("""mesh {K:4}

func @main(%x: tensor<2x2xf32>) -> tensor<2x2xf32> {
  %r = all_reduce ["K"] %x : tensor<2x2xf32>
  return %r
}
""", None),
    "divergent": ("""mesh {K:2}

func @main(%x: tensor<4x4xf32>) -> tensor<2x4xf32> {
  %s = all_slice [["K"], []] %x : tensor<2x4xf32>
  return %s
}
""", None),
}

ACCEPTANCE = {
    "chain": (["bp"], ["mp"], ["bp", "mp"], ["bp", "mp", "z3"]),
    "mlp": (["bp"], ["mp"], ["bp", "mp"], ["bp", "z2"], ["bp", "z3"],
            ["bp", "mp", "z2"], ["bp", "mp", "z3"], ["es"], ["bp", "es"]),
    "transformer": (["bp"], ["mp"], ["bp", "mp"], ["bp", "mp", "z2"], ["bp", "mp", "z3"]),
    "transpose_diag": (["tp"], ["tp_unresolved"]),
}

EMB = ("E", {"x": 1, "y": 1})
STEPS = [
    # name, model, params, mesh, stages, extra tactics, scale, seeds
    ("mlp1_bp_B2", "mlp", dict(hidden_layers=1, batch=64, width=48), "B:2", ["bp"], [], 0.25, [0, 1]),
    ("mlp2_bpz3_B4", "mlp", dict(hidden_layers=2, batch=32, width=32), "B:4", ["bp", "z3"], [], 0.25, [0]),
    ("tf2_bpmp_B2M2", "transformer", dict(blocks=2, batch=32, d_model=32, d_ff=64), "B:2,M:2",
     ["bp", "mp"], [], 0.1, [0, 1]),
    ("tf2_bpz3_B4", "transformer", dict(blocks=2, batch=32, d_model=32, d_ff=64), "B:4",
     ["bp", "z3"], [], 0.1, [0]),
    ("tf1_bpmpz3emb_B2M2E2", "transformer", dict(blocks=1, batch=32, d_model=32, d_ff=64),
     "B:2,M:2,E:2", ["bp", "mp", "z3"], [EMB], 0.1, [0, 1]),
    ("tf2_bpmpz2_B2M2", "transformer", dict(blocks=2, batch=32, d_model=32, d_ff=64), "B:2,M:2",
     ["bp", "mp", "z2"], [], 0.1, [0]),
    # C4 U-Net analog (tools/unet_model.py): 1x1-conv encoder/decoder with pool,
    # upsample and skip -- rank-6 reshape/reduce/broadcast in the local program
    ("unet_bp_B2", "unet", dict(batch=4, height=4, width=4, c0=4, c1=8, c2=8), "B:2", ["bp"], [], 0.25, [0]),
    ("unet_bpz2_B4", "unet", dict(batch=4, height=4, width=4, c0=4, c1=8, c2=8), "B:4", ["bp", "z2"], [],
     0.25, [0, 1]),
]


def replicated_spec(func):
    return ShardingSpec(args={n: [[] for _ in t.dims] for n, t in func.args},
                        results=[[[] for _ in t.dims] for t in func.result_types])


def op_sites():
    T = TensorType
    yield "matmul_4x8x2", "matmul", [T((4, 8)), T((8, 2))], {}
    yield "matmul_5x7x3", "matmul", [T((5, 7)), T((7, 3))], {}
    yield "matmul_64x48x80", "matmul", [T((64, 48)), T((48, 80))], {}
    yield "add", "add", [T((6, 10)), T((6, 10))], {}
    yield "mul", "mul", [T((6, 10)), T((6, 10))], {}
    yield "neg", "neg", [T((3, 5))], {}
    yield "exp", "exp", [T((3, 5))], {}
    yield "tag", "tag", [T((4, 4))], {"name": "t"}
    yield "transpose2", "transpose", [T((4, 12))], {"perm": [1, 0]}
    yield "transpose3", "transpose", [T((4, 8, 12))], {"perm": [2, 0, 1]}
    yield "reduce0", "reduce", [T((12, 8))], {"dims": [0]}
    yield "reduce1max", "reduce", [T((12, 8))], {"dims": [1], "monoid": "max"}
    yield "reduce02", "reduce", [T((4, 8, 12))], {"dims": [0, 2]}
    yield "reduce01", "reduce", [T((12, 8))], {"dims": [0, 1]}
    yield "reduce0max3", "reduce", [T((5, 6, 7))], {"dims": [1], "monoid": "max"}
    yield "reshape1", "reshape", [T((4, 8))], {"dims": (32,)}
    yield "reshape2", "reshape", [T((4, 8, 12))], {"dims": (32, 12)}
    yield "reshape3", "reshape", [T((4, 8))], {"dims": (4, 2, 4)}
    yield "broadcast1", "broadcast", [T((8,))], {"dims": [1], "shape": (4, 8)}
    yield "broadcast2", "broadcast", [T((4, 8))], {"dims": [0, 2], "shape": (4, 4, 8)}
    yield "broadcast0", "broadcast", [T((8,))], {"dims": [0], "shape": (8, 3)}


def main():
    cases, arrays = [], {}

    def put(key, arr):
        arrays[key] = np.asarray(arr)

    # --- A: hand-written collective programs -------------------------------
    for name, (text, layouts) in RULE_PROGRAMS.items():
        for variant in ("raw", "fused"):
            m = parse_module(text)
            if variant == "fused":
                fuse_collectives(m.func("main"))
                if print_module(m) == print_module(parse_module(text)):
                    continue
            spec = replicated_spec(m.func("main"))
            if layouts is not None:
                spec.results = layouts
            rng = np.random.default_rng(7)
            if name == "ones_ar":
                ins = {"x": np.ones((2, 2), np.float32)}
                recipe = {"kind": "ones"}
            elif name == "divergent":
                ins = {"x": np.arange(16.0, dtype=np.float32).reshape(4, 4)}
                recipe = {"kind": "arange"}
            else:
                ins = {n: rng.standard_normal(t.dims).astype(np.float32)
                       for n, t in m.func("main").args}
                recipe = {"kind": "normal", "seed": 7}
            key = f"rule_{name}_{variant}"
            case = {"key": key, "group": "rule", "local_ir": print_module(m),
                    "sharding": spec.to_json(), "inputs": recipe, "seeds": [0],
                    "counts": collective_counts(m)}
            try:
                outs = spmd_interpret(m, spec, ins)
                for j, o in enumerate(outs):
                    put(f"{key}/s0/spmd/{j}", o)
                case["n_out"] = len(outs)
            except DivergenceError as e:
                case["error"] = "DivergenceError"
                case["error_text"] = str(e)
            cases.append(case)

    # --- B: acceptance matrix at the reference's toy sizes -----------------
    for model, schedules in ACCEPTANCE.items():
        mesh = "M:2" if model == "transpose_diag" else "B:4,M:2"
        for names in schedules:
            module = build_model(model)
            module.mesh = Mesh.parse(mesh)
            p = Partitioner(module)
            for t in cookbook_schedule(model, names, module):
                p.apply(t)
            base = parse_module(p.base_ir)
            loc, spec = localize(lower_to_spmd(p.module))
            key = f"acc_{model}_{'+'.join(names)}"
            case = {"key": key, "group": "acceptance", "dense_ir": p.base_ir,
                    "local_ir": print_module(loc), "sharding": spec.to_json(),
                    "inputs": {"kind": "random_inputs", "scale": 0.25}, "seeds": [0, 1],
                    "counts": collective_counts(loc),
                    "compute_flops": simulate(loc, BUILTIN_SPECS["tpu-v3-core"]).compute_flops}
            for s in case["seeds"]:
                ins = random_inputs(base, seed=s)
                want = interpret(base, ins)
                got = spmd_interpret(loc, spec, ins, tol=1e-5)
                for j, (g, w) in enumerate(zip(got, want)):
                    put(f"{key}/s{s}/spmd/{j}", g)
                    put(f"{key}/s{s}/dense/{j}", w)
                case["n_out"] = len(got)
            cases.append(case)

    # --- C: small training steps with the benchmark configs' structure -----
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(HERE)), "tools"))
    from unet_model import unet_schedule, unet_train
    for name, model, params, mesh, stages, extra, scale, seeds in STEPS:
        module = unet_train(**params) if model == "unet" else build_model(model, **params)
        module.mesh = Mesh.parse(mesh)
        p = Partitioner(module)
        tactics = (unet_schedule(stages, module) if model == "unet"
                   else cookbook_schedule(model, stages, module))
        for t in tactics:
            p.apply(t)
        for ax, s in extra:
            p.apply(ManualPartition(ax, dict(s)))
        base = parse_module(p.base_ir)
        loc, spec = localize(lower_to_spmd(p.module))
        key = f"step_{name}"
        case = {"key": key, "group": "step", "dense_ir": p.base_ir,
                "local_ir": print_module(loc), "sharding": spec.to_json(),
                "inputs": {"kind": "random_inputs", "scale": scale}, "seeds": seeds,
                "counts": collective_counts(loc),
                "compute_flops": simulate(loc, BUILTIN_SPECS["tpu-v3-core"]).compute_flops}
        for s in seeds:
            ins = random_inputs(base, seed=s, scale=scale)
            want = interpret(base, ins)
            got = spmd_interpret(loc, spec, ins, tol=1e-5)
            for j, (g, w) in enumerate(zip(got, want)):
                assert np.all(np.isfinite(w)), (name, j)
                put(f"{key}/s{s}/spmd/{j}", g)
                put(f"{key}/s{s}/dense/{j}", w)
            case["n_out"] = len(got)
        cases.append(case)

    # --- D: one-op dense programs ------------------------------------------
    for name, kind, types, attrs in op_sites():
        b = FuncBuilder()
        names = [b.arg(f"a{i}", t.dims, t.elem) for i, t in enumerate(types)]
        r = b.emit(kind, names, dict(attrs))
        b.ret(r)
        m = b.build()
        key = f"op_{name}"
        case = {"key": key, "group": "op", "dense_ir": print_module(m),
                "inputs": {"kind": "random_inputs", "scale": 1.0}, "seeds": [0], "n_out": 1}
        ins = random_inputs(m, seed=0, scale=1.0)
        (out,) = interpret(m, ins)
        put(f"{key}/s0/dense/0", out)
        cases.append(case)

    # pin the input generator itself: a fingerprint of one draw
    fp = random_inputs(build_model("mlp"), seed=3)
    put("fingerprint/random_inputs_mlp_s3/x", fp["x"])

    with open(os.path.join(HERE, "cases.json"), "w") as fh:
        json.dump(cases, fh, indent=0)
    np.savez_compressed(os.path.join(HERE, "outputs.npz"), **arrays)
    print(f"{len(cases)} cases, {len(arrays)} arrays, "
          f"{sum(a.nbytes for a in arrays.values()) / 1e6:.2f} MB raw")


if __name__ == "__main__":
    main()
