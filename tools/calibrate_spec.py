"""Calibrate a B200 MachineSpec for the reference's simulator from the
measured bench lines.

The reference costs a localized program as
    runtime = compute_flops / peak_flops + sum_collectives(bytes / link_bandwidth + latency)
(`simulate`, sim.py:209-234; ring bytes `collective_bytes`, sim.py:114-123).
This tool extracts, per measured program, the simulator's own inputs (F, the
per-collective ring bytes and the collective count), fits
    * peak_flops from the N=1 transformer steps (compute only),
    * link_bandwidth and collective_latency_s (non-negative least squares) from
      the multi-GPU residuals,
writes the spec in the reference's `key = value` format
(`parse_machine_spec`, sim.py:47-74) and prints simulated vs measured step
times.  Runs where the reference is importable (this container):

    PYTHONPATH=/root/reference/pkg/src python tools/calibrate_spec.py
"""
import glob
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT_SPEC = os.path.join(ROOT, "paper_2401_11202_b200", "machine", "b200-spindle.spec")


def sim_inputs(prog_name):
    from spindle.parser import parse_module
    from spindle.sim import collective_bytes, _flops
    d = os.path.join(ROOT, "paper_2401_11202_b200", "programs", prog_name)
    meta = json.load(open(os.path.join(d, "meta.json")))
    path = os.path.join(d, "local.ir" if meta.get("mesh") else "dense.ir")
    m = parse_module(open(path).read())
    if meta.get("mesh") and m.mesh is None:
        from spindle.ir import Mesh
        m.mesh = Mesh.parse(meta["mesh"])
    f = m.func("main")
    types = {n: t for n, t in f.args}
    F, B, n = 0.0, 0.0, 0
    for op in f.ops:
        for r, t in zip(op.results, op.result_types):
            types[r] = t
        if op.kind in ("all_gather", "all_reduce", "reduce_scatter", "all_to_all"):
            B += collective_bytes(op, m.mesh, types[op.operands[0]].nbytes)
            n += 1
        elif op.kind != "all_slice":
            F += _flops(op, [types[o].dims for o in op.operands])
    return F, B, n


def bench_lines(rnd):
    """(tag, bench JSON line) of round `rnd`'s committed measurements."""
    out = []
    if rnd == 1:
        for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r01_bench_c*_n*.json"))):
            if "first" in path or "reference" in path:
                continue
            out.append((os.path.basename(path)[10:-5], json.load(open(path))))
        return out
    # round 2: the N=1 lines and the final N=2/4 lines of one 4-GPU box
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r02_bench_c*_n1.json"))):
        if "reference" in path:
            continue
        line = json.loads(open(path).read().strip().splitlines()[-1])
        out.append((os.path.basename(path)[10:-5], line))
    for raw in open(os.path.join(ROOT, "profiles", "r02_scale_final_lines.jsonl")):
        raw = raw.strip()
        if raw.startswith("{"):
            line = json.loads(raw)
            cfg = line["config"].get("config") or line["config"]["program"][:2]
            out.append((f"{cfg}_n{line['n_gpus']}", line))
    return out


def main():
    rnd = 2 if "--round" not in sys.argv else int(sys.argv[sys.argv.index("--round") + 1])
    rows = []
    for tag, line in bench_lines(rnd):
        prog = line["config"]["program"]
        if prog.startswith("c1"):
            continue                 # launch-bound toy step: no information on peak or links
        F, B, n = sim_inputs(prog)
        rows.append(dict(cfg=tag, prog=prog, N=line["n_gpus"], t=line["ms_per_step"] / 1e3, F=F, B=B, n=n))
    # peak: N=1 transformer steps (the simulator has no HBM term; C4's
    # memory-bound U-Net is reported but not fitted)
    fit1 = [r for r in rows if r["N"] == 1 and not r["cfg"].startswith("c4")]
    peak = sum(r["F"] for r in fit1) / sum(r["t"] for r in fit1)
    # link bandwidth + latency: NNLS on residuals of the multi-GPU transformer runs
    fitn = [r for r in rows if r["N"] > 1 and not r["cfg"].startswith("c4")]
    A = np.array([[r["B"], r["n"]] for r in fitn])
    y = np.array([max(0.0, r["t"] - r["F"] / peak) for r in fitn])
    best = None
    for lat in np.linspace(0, 50e-6, 501):
        rhs = y - A[:, 1] * lat
        inv_bw = max(1e-15, float(A[:, 0] @ rhs / (A[:, 0] @ A[:, 0])))
        err = float(np.sum((A[:, 0] * inv_bw + A[:, 1] * lat - y) ** 2))
        if best is None or err < best[0]:
            best = (err, inv_bw, lat)
    _, inv_bw, lat = best
    bw = 1.0 / inv_bw
    os.makedirs(os.path.dirname(OUT_SPEC), exist_ok=True)
    with open(OUT_SPEC, "w") as fh:
        fh.write("# B200 running the spindle_b200 evaluator (fp32 semantics, block-scaled 3xFP16\n"
                 f"# tensor-core GEMMs), calibrated by tools/calibrate_spec.py from round {rnd}'s bench lines.\n"
                 "# peak_flops: effective f32 rate of whole N=1 transformer steps (all ops);\n"
                 "# link_bandwidth / collective_latency_s: fitted to the multi-GPU residuals\n"
                 "# (collectives partly overlap compute here, so these are effective values).\n"
                 "name = b200-spindle\n"
                 f"peak_flops = {peak:.4e}\n"
                 "hbm_bytes = 1.8e11\n"
                 f"link_bandwidth = {bw:.4e}\n"
                 f"collective_latency_s = {lat:.2e}\n")
    from spindle.sim import load_machine_spec
    spec = load_machine_spec(OUT_SPEC)
    print(f"spec: peak_flops {spec.peak_flops:.3e}  link_bandwidth {spec.link_bandwidth:.3e}  "
          f"collective_latency_s {spec.collective_latency_s:.2e}  ({OUT_SPEC})")
    print(f"{'config':8s} {'N':>2s} {'program':26s} {'measured ms':>12s} {'simulated ms':>13s} {'error':>7s}")
    for r in rows:
        sim = r["F"] / spec.peak_flops + r["B"] / spec.link_bandwidth + r["n"] * spec.collective_latency_s
        print(f"{r['cfg']:8s} {r['N']:2d} {r['prog']:26s} {r['t'] * 1e3:12.3f} {sim * 1e3:13.3f} "
              f"{100 * (sim - r['t']) / r['t']:+6.1f}%")


if __name__ == "__main__":
    main()
