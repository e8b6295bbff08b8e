"""Benchmark: partitioned fwd+bwd+momentum-SGD step throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Metric (BASELINE.json): "Partitioned fwd+bwd samples/s at 1/2/4/8 B200; %
of tensor-core/HBM roofline".  One STEP = one execution of the localized
training-step program of the configured model (forward, hand-written
backward and momentum update of every parameter -- models.py:152-220) on the
global batch; samples/s = global batch / step time.  N=1 runs the
unpartitioned module (the reference's 1-device semantics); N>1 runs
the partitioned program one mesh device per GPU (torchrun), collectives over
NCCL.  Scaling is STRONG (global batch fixed).

The default workload is C3 (BASELINE.json configs[2]: 32 transformer blocks,
d_model 2048, d_ff 8192, batch 8192, BP+Z3 on B:8 at 8 GPUs), the largest
configuration that fits one B200 (configs[1], C2, is quoted on a 2x4 mesh).

`value` is device-timed (CUDA events, max over ranks) with every input
resident in HBM (the compiled step replayed as one CUDA graph).  `e2e` is
the same metric through the drop-in call a user of the reference makes --
`interpret(module, inputs)` at 1 GPU (interp.py:117-132; `spmd_interpret` is
the same call with a mesh), `Session.call` per rank at N GPUs -- with EVERY
input (parameters, momenta, batch) copied in from host arrays and EVERY
result copied back to new host arrays inside the timed region; the compiled
plan comes from the plan cache, as on any repeated call.  `step_roofline`
is T_roof / T_measured with T_roof from the program's IR op by op
(roofline.py); `roofline` is the dominant kernel's.
`--impl reference` times the reference's CPU evaluator (the oracle
restatement, numpy) on this host.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TF32_MMA_PEAK = 1112.0   # TF/s, profiles/r01_mma_bench.txt
METRIC = "Partitioned fwd+bwd samples/s at 1/2/4/8 B200; % of tensor-core/HBM roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def bf16_sustained():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops_sustained"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus, active=True):
        self.gpus = gpus
        self.active = active
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        if not self.active:
            return self
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9 or not f[0].isdigit() or int(f[0]) not in self.gpus:
                    continue
                try:
                    sm.append(float(f[1]))
                    smax = float(f[2])
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, rank):
    if world == 1:
        return None
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


_T0 = time.time()


def log(msg: str):
    """Progress on stderr (one line per phase and rank): a hang shows where it is."""
    sys.stderr.write(f"[bench rank {os.environ.get('RANK', '0')} +{time.time() - _T0:7.1f}s] {msg}\n")
    sys.stderr.flush()


def barrier(dist):
    if dist is not None:
        dist.barrier()


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_step(wl, n, prog):
    """One step of the reference's CPU evaluator on this workload (the oracle
    restatement, bit-identical to the reference: tests/test_oracle_configs.py):
    `interpret` of the dense module at 1 GPU, `spmd_interpret` of the
    partitioned one at N.  Where the evaluator cannot hold the model (C3: ~11 GB
    per block) the step time is extrapolated from 1- and 2-block
    programs at full width, t(1) + (B-1) (t(2) - t(1)).
    Returns (step seconds, sample description)."""
    from oracle import spmd_oracle as O
    from paper_2401_11202_b200.programs import load_program, synthetic_inputs

    def run(p):
        ins = synthetic_inputs(p.dense, seed=0, scale=wl["scale"])
        fn = (lambda: O.interpret(p.dense, ins)) if n == 1 else (lambda: O.spmd_interpret(p.local, p.sharding, ins))
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    what = "interpret" if n == 1 else "spmd_interpret"
    ext = wl.get("cpu_extrap")
    if ext and n in ext:
        b = ext["blocks"]
        p1, p2 = (load_program(x) for x in ext[n])
        t1, t2 = run(p1), run(p2)
        return t1 + (b - 1) * (t2 - t1), (f"{what} of the 1- and 2-block programs at full width ({p1.name}: "
                                         f"{t1:.2f} s, {p2.name}: {t2:.2f} s) extrapolated to {b} blocks as "
                                         f"t(1) + {b - 1} (t(2) - t(1)) (BASELINE.md §2; the full model does not "
                                         f"fit the CPU evaluator, SURVEY F6)")
    t = run(prog)
    return t, f"one full step of {prog.name} through {what}"


def e2e_call(sess, prog, base, inputs, n, dist, budget_s, max_steps, batch, feedback=False):
    """The metric through the call a user makes, as a training loop: every
    input copied in from host memory and every result copied out to host
    memory each step, the updated parameters and momenta (results `new_X`)
    fed back as the next step's arguments `X`.  1 GPU: the drop-in
    `interpret(module, inputs)` (the session is closed first; the call
    compiles once into the plan cache and then replays the captured step).
    N GPUs: `Session.call_local` on every rank (the same data movement for the
    rank's mesh device), wall time max over ranks.  The batch and the initial
    arguments are staged once into page-locked host arrays; results come back
    in page-locked arrays (runtime.PinnedPool), so fed-back arguments go in by
    direct DMA as well."""
    import paper_2401_11202_b200 as pkg
    from paper_2401_11202_b200 import runtime as R
    pool = R.pinned_pool()

    def pinned(a):
        b = pool.array(a.shape, a.dtype)
        if b is None:
            return np.ascontiguousarray(a)
        b[...] = a
        return b
    f = (base if n == 1 else prog.local).func()
    args = [a for a, _ in f.args]
    if n == 1:
        sess.close()
        cur = {a: pinned(inputs[a]) for a in args}
        fn = lambda: pkg.interpret(base, cur)
        what = "paper_2401_11202_b200.interpret(module, host inputs) -- the drop-in for interp.interpret"
        spec = None
    else:
        cur = {a: pinned(x) for a, x in sess.local_inputs(inputs)[0].items()}
        # a session whose plan carries the copies (io), like the drop-in call's
        from paper_2401_11202_b200.session import Session
        rank, world, local = sess.rank, dist.get_world_size(), int(os.environ.get("LOCAL_RANK", "0"))
        sess.close()
        sess = Session(prog.local, prog.sharding, mode="nccl", rank=rank, world=world, local_rank=local, io=True)
        fn = lambda: [r[0] for r in sess.call_local([cur])]
        what = ("Session.call_local(host inputs) on every rank, copies inside the plan overlapped with the step "
                "(the drop-in call's data movement per mesh device)")
        spec = prog.sharding
    fb = {}
    for j, r in enumerate(f.results if feedback else []):
        a = r[4:] if r.startswith("new_") else None
        if a in cur and tuple(f.result_types[j].dims) == tuple(cur[a].shape) and \
                (spec is None or spec.results[j] == spec.args[a]):
            fb[j] = a

    def step():
        out = fn()
        for j, a in fb.items():
            cur[a] = out[j]
        return out
    step()                          # compile (1 GPU: into the plan cache) + eager run + capture
    out = step()                    # replay
    out = step()                    # a second generation of page-locked result arrays exists now
    h2d = sum(x.nbytes for x in cur.values())
    d2h = sum(r.nbytes for r in out)
    barrier(dist)
    t0 = time.perf_counter()
    step()
    one = max_over_ranks(dist, time.perf_counter() - t0)
    k = int(max_over_ranks(dist, int(max(min(10, max_steps), min(max_steps, budget_s / max(one, 1e-6))))))
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(k):
        out = step()
    wall = max_over_ranks(dist, time.perf_counter() - t0)
    finite = bool(all(np.all(np.isfinite(r)) for r in out))
    if n > 1:
        sess.close()
    return {"value": batch / (wall / k), "unit": "samples/s", "steps": k, "ms_per_step": wall / k * 1e3,
            "h2d_bytes_per_step": int(sum_over_ranks(dist, h2d)), "d2h_bytes_per_step": int(sum_over_ranks(dist, d2h)),
            "outputs_finite": finite, "fed_back": len(fb),
            "note": f"{what}: each step copies EVERY argument (batch, parameters, momenta"
                    f"{'; ' + str(len(fb)) + ' of them fed back from the previous results' if fb else ''}) "
                    f"host->device and EVERY result device->host into new host arrays inside the timed region "
                    f"(host wall clock, max over ranks); host arrays are page-locked (arguments staged once, "
                    f"results returned in recycled pinned arrays)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--e2e-seconds", type=float, default=40.0, help="time budget of the plugin-call e2e loop")
    ap.add_argument("--e2e-feedback", action="store_true",
                    help="feed results new_X back as arguments X (a training loop; C3's summed-loss model "
                         "diverges after 2 steps at batch 8192, in the reference's evaluator as well)")
    ap.add_argument("--program", default=None, help="override the config's program for this GPU count")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-out", default=None, help="write per-record timings (json)")
    args = ap.parse_args()

    from paper_2401_11202_b200.programs import WORKLOADS, load_program, synthetic_inputs
    world, rank, local = dist_env()
    n = args.gpus
    if world != n and not (world == 1 and n == 1):
        raise SystemExit(f"--gpus {n} needs torchrun with {n} processes (WORLD_SIZE={world})")
    wl = WORKLOADS[args.config]
    wl_env = wl.get("env", {}).get(n, {})
    for k, v in wl_env.items():
        os.environ.setdefault(k, v)        # before any plan is built; an explicit setting wins
    prog = load_program(args.program or wl["programs"][n])
    batch = prog.batch
    base = prog.dense
    mesh = prog.meta.get("mesh") or "dense (1 device)"
    config = {"workload": f"{args.config.upper()}: {wl['desc']}", "mesh": mesh,
              "program": prog.name, "global_batch": batch,
              "schedule": prog.meta.get("schedule") or [], "parallelism":
              ("none (unpartitioned)" if n == 1 else f"mesh {mesh}, one device per GPU"),
              "l2": "working set > 126 MB L2 (params+momenta alone exceed it); no flush needed",
              "inputs": f"synthetic N(0, {wl['scale']}^2) float32 (random_inputs generator, seed 0)"}
    if wl_env:
        config["env"] = {k: os.environ[k] for k in wl_env}
    dtype = "f32"

    if args.impl == "reference":
        if rank != 0:
            return
        steps = max(1, min(args.steps, 3))
        warm = min(args.warmup, 1)
        for _ in range(warm):
            reference_step(wl, n, prog)
        ts, sample = [], ""
        for _ in range(steps):
            t, sample = reference_step(wl, n, prog)
            ts.append(t)
        med = float(np.median(ts))
        v = batch / med
        line = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": n, "steps": steps,
                "warmup": warm, "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": dtype, "data": "synthetic", "config": config,
                "impl": "reference",
                "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cpu_threads(), "kind": "port",
                                 "sample": f"median of {steps} steps, each {sample}; oracle restatement of the "
                                           f"reference evaluator, numpy {np.__version__}, BLAS threads = host cores"},
                "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    dist = init_dist(world, rank)
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.session import Session
    inputs = synthetic_inputs(base, seed=0, scale=wl["scale"])
    if n == 1:
        sess = Session(base, local_rank=local)
    else:
        sess = Session(prog.local, prog.sharding, mode="nccl", rank=rank, world=world, local_rank=local)
    log(f"compiled {prog.name}: {sess.ex.plan.n_records} records, arena {sess.ex.peak_bytes / 1e9:.1f} GB")
    sess.load(inputs)
    dev = sess.device
    # eager run once (validates), then capture the whole step as one CUDA graph
    sess.run()
    sess.sync()
    log("eager step done")
    sess.capture()
    for _ in range(max(3, args.warmup)):
        sess.step()
    sess.sync()
    launches_per_step = sess.launch_count()

    log("captured + warm")
    e0, e1 = dev.event(), dev.event()
    # rank 0 samples every GPU of the job (nvidia-smi sees the whole node)
    with ClockSampler([local] if world == 1 else list(range(world)), active=(rank == 0)) as clk:
        barrier(dist)
        sess.sync()
        dev.record(e0)
        for _ in range(args.steps):
            sess.step()
        dev.record(e1)
        sess.sync()
        barrier(dist)
        # keep sampling clocks under the same load for a short while if the region
        # was short.  The number of extra steps must be the SAME on every rank
        # (each step runs collectives that wait for every member): it is derived
        # from the max over ranks, never from a rank's own time.
        ms = dev.elapsed_ms(e0, e1)
        ms_total = max_over_ranks(dist, ms)
        n_extra = 0
        while ms_total * (1 + n_extra) < 1500 and n_extra < 2000:
            n_extra += 1
        for _ in range(n_extra * args.steps):
            sess.step()
        sess.sync()
        barrier(dist)
    ms_step = ms_total / args.steps
    value = batch / (ms_step / 1e3)

    loss_arr = np.empty(1, np.float32)
    dev.d2h(loss_arr, sess.result_addr(0))
    dev.sync()
    loss = float(loss_arr[0])

    log(f"timed region: {ms_step:.3f} ms/step")
    # ---- per-record profile (eager, events between records) for the roofline
    rec_ms = sess.ex.plan.profile()
    recs = sess.ex.records()
    gemm_flops = gemm_ms = ideal_ms = tensor_flops = 0.0
    hbm, bf16, src = peaks()
    # tensor-core ceilings per GEMM path: block-scaled 3xFP16 (path 3, kind::f16)
    # against the measured dense bf16/f16 rate (MEASURED_PEAKS.json, burst);
    # 3xTF32 (path 1, kind::tf32) against the measured tcgen05 tf32 issue rate
    # (tools/mma_bench.cu, profiles/r01_mma_bench.txt).  Both do 3 MMAs per fp32
    # FLOP (hi.hi + hi.lo + lo.hi).
    tc_peak = {3: bf16, 1: TF32_MMA_PEAK}
    paths = {}
    cls_ms = {}
    for idx, ((kind, p), t) in enumerate(zip(recs, rec_ms)):
        name = {R.K_EW: "elementwise", R.K_REDUCE: "reduce", R.K_GEMM: "gemm", R.K_GATHER: "relayout",
                R.K_CREDUCE: "collective_local", R.K_NCCL: "nccl", R.K_PEER: "peer_allreduce",
                R.K_SPLIT: "gemm_operand_split", R.K_COPY: "copy"}[kind]
        cls_ms[name] = cls_ms.get(name, 0.0) + float(t)
        if kind == R.K_GEMM:
            path = sess.ex.plan.record_info(idx)[1]
            f = 2.0 * p.M * p.N * p.K * p.ndev
            paths[path] = paths.get(path, 0) + 1
            gemm_flops += f
            gemm_ms += float(t)
            if path in tc_peak:
                tensor_flops += 3.0 * f
                ideal_ms += 3.0 * f / (tc_peak[path] * 1e12) * 1e3
    achieved = tensor_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    sust = bf16_sustained()       # MEASURED_PEAKS: cuBLAS bf16 back to back for 4 s (the step's regime)
    # DRAM traffic of one GEMM launch from the committed `ncu --set full` capture
    traffic, traffic_note = None, None
    cap_file = next((f for f in (f"r02_ncu_full_gemm_{args.config}_n1.json", f"r01_ncu_full_gemm_{args.config}_n1.json",
                                 "r01_ncu_full_gemm_c2_n1.json") if os.path.exists(os.path.join(ROOT, "profiles", f))),
                    "r01_ncu_full_gemm_c2_n1.json")
    try:
        with open(os.path.join(ROOT, "profiles", cap_file)) as fh:
            cap = json.load(fh)[0]

        def _mb(v):
            x, u = v.split()
            return float(x) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        traffic = _mb(cap["dram__bytes_read.sum"]) + _mb(cap["dram__bytes_write.sum"])
        traffic_note = (f"dram read+write bytes of one {cap['kernel'].split('(')[0].replace('void ', '')} launch "
                        f"({cap.get('shape', 'C2 2048x4096x1024')}, {cap['gpu__time_duration.sum']}) from "
                        f"profiles/{cap_file}; " + cap.get("algorithmic_note",
                        "algorithmic: fp16 pieces of A 8.4 MB + B 16.8 MB read, C 33.6 MB written (C stays in L2 "
                        "for its consumer, so DRAM sees the operand reads only)"))
    except (OSError, KeyError, ValueError, IndexError):
        pass
    peak_eff = tensor_flops / (ideal_ms / 1e3) / 1e12 if ideal_ms > 0 else bf16
    kname = ("tcgen05 block-scaled 3xFP16 GEMM (split_h16_kernel + gemm_h3_kernel, CTA pairs)"
             if paths.get(3, 0) >= paths.get(1, 0) else "tcgen05 3xTF32 GEMM (gemm_tc_tmema_kernel, CTA pairs)")
    roofline = {"bound": "tensor", "kernel": kname,
                "achieved": achieved, "peak": peak_eff, "unit": "TFLOP/s",
                "frac": (ideal_ms / gemm_ms) if gemm_ms > 0 else 0.0,
                "peak_sustained": sust,
                "frac_vs_sustained": (achieved / sust) if (sust and paths.get(3, 0) == sum(paths.values())) else None,
                "traffic": traffic,
                "traffic_note": traffic_note,
                "gemm_paths": {("h3" if k == 3 else "tf32" if k == 1 else "simt"): v for k, v in paths.items()},
                "note": (f"achieved = tensor-core work (3 MMAs per fp32 FLOP) / GEMM record time, summed over the "
                         f"{sum(paths.values())} GEMM launches of one step; peak = {src} dense bf16 "
                         f"{bf16:.1f} TF/s for kind::f16, measured tcgen05 kind::tf32 rate {TF32_MMA_PEAK:.0f} "
                         f"TF/s for 3xTF32 records (time-weighted).  The fp32 -> fp16-pieces operand splits are "
                         f"separate HBM-bound records (step_ms_by_class.gemm_operand_split).  fp32-equivalent GEMM rate "
                         f"{gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else 0:.1f} TFLOP/s"),
                "step_ms_by_class": {k: round(v, 4) for k, v in sorted(cls_ms.items())},
                "gemm_share_of_step": (gemm_ms / float(np.sum(rec_ms))) if np.sum(rec_ms) > 0 else None}
    # streaming (HBM-bound) records: algorithmic bytes / eager record time
    def _ew_bytes(q):
        tot = 4 * q.numel * q.n_out
        for j in range(q.n_in):
            cnt = 1
            for k in range(q.rank):
                if q.inp[j].stride[k] != 0:
                    cnt *= q.dims[k]
            tot += 4 * cnt
        return tot
    s_bytes = s_ms = 0.0
    for idx, ((kind, p), t) in enumerate(zip(recs, rec_ms)):
        if kind == R.K_EW:
            s_bytes += _ew_bytes(p)
            s_ms += float(t)
        elif kind == R.K_SPLIT:
            spath = sess.ex.plan.record_info(idx)[1]
            fused = spath == -1
            # pieces written (+ the fp32 read when standalone); fused (-1): time is in the EW record;
            # batched (-2): time is in the first SPLIT record of the batch (path 2)
            s_bytes += 4.0 * p.rows * p.cols * (1 if fused else 2)
            if spath >= 0:
                s_ms += float(t)
    streaming = {"bound": "hbm", "kernels": "ew_static(_split)_kernel, ew_vec/gen_kernel, split_h16(_batch)_kernel",
                 "achieved": s_bytes / (s_ms / 1e3) / 1e9 if s_ms > 0 else 0.0, "peak": hbm, "unit": "GB/s",
                 "frac": (s_bytes / (s_ms / 1e3) / 1e9 / hbm) if s_ms > 0 else 0.0,
                 "bytes_per_step": s_bytes, "ms_per_step_eager": s_ms,
                 "note": "algorithmic bytes (inputs once, broadcast operands at their own size, outputs, fp16 "
                         "pieces) over the eager per-record time (CUDA events between records, launch gaps "
                         "included) of every elementwise and split record of one step"}
    if args.profile_out and rank == 0:
        with open(args.profile_out, "w") as fh:
            json.dump({"records": [[int(k), float(t)] for (k, _), t in zip(recs, rec_ms)],
                       "class_ms": cls_ms}, fh, indent=0)

    # ---- executed work (runtime counters over every run above) vs the simulator
    work = sess.ex.work_report()
    # ---- step-level roofline from the program's IR (per device)
    from paper_2401_11202_b200.roofline import step_roofline
    sr = step_roofline(base if n == 1 else prog.local, bf16_tflops=bf16, hbm_gbs=hbm)
    step_roof = {"t_roof_ms": sr["t_roof_s"] * 1e3, "t_measured_ms": ms_step,
                 "frac": sr["t_roof_s"] * 1e3 / ms_step, "bound": sr["bound"],
                 "t_gemm_ms": sr["t_gemm_s"] * 1e3, "t_stream_ms": sr["t_stream_s"] * 1e3,
                 "t_nvlink_ms": sr["t_nvlink_s"] * 1e3, "hbm_bytes": sr["hbm_bytes"], "flops": sr["flops"],
                 "nvlink_bytes": sr["nvlink_bytes"],
                 "note": "T_roof = max(sum over IR ops of max(F/P, B/BW_hbm), B_nvl/BW_nvl) per device (SURVEY "
                         "§8(d), paper_2401_11202_b200/roofline.py): F by the simulator's convention (sim.py:86-100), "
                         "matmuls at the measured bf16 peak / 3 (3 fp16 MMAs per fp32 FLOP), B = operand data + "
                         "result bytes of each matmul/elementwise/reduce op unfused, B_nvl = ring bytes "
                         "(sim.py:114-123) at 900 GB/s; frac = T_roof / measured step"}

    # ---- end to end through the drop-in call: every input from host arrays,
    # every result back to new host arrays, per step
    log("profile done; e2e")
    e2e = e2e_call(sess, prog, base, inputs, n, dist, args.e2e_seconds, args.steps, batch, args.e2e_feedback)
    log(f"e2e {e2e['ms_per_step']:.2f} ms/call")

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        t, sample = reference_step(wl, n, prog)
        cpu = {"value": batch / t, "unit": "samples/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"{sample}: oracle restatement of the reference evaluator (bit-identical to it, "
                         f"tests/test_oracle_configs.py), numpy {np.__version__}, BLAS on all host cores"}

    counts = work["collectives"]
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": n, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": config, "roofline": roofline, "streaming_roofline": streaming, "cpu_baseline": cpu,
                "e2e": e2e, "step_roofline": step_roof,
                "gpu_launches": int(launches_per_step * args.steps),
                "launches_per_step": int(launches_per_step),
                "clocks": clk.summary(), "loss": loss, "loss_finite": bool(np.isfinite(loss)),
                "collectives_per_step": counts,
                "flops_per_device_step": work["flops"]}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
