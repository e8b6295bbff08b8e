"""Benchmark: partitioned fwd+bwd+momentum-SGD step throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Metric (BASELINE.json): "Partitioned fwd+bwd samples/s at 1/2/4/8 B200; %
of tensor-core/HBM roofline".  One STEP = one execution of the localized
training-step program of the configured model (forward, hand-written
backward and momentum update of every parameter -- models.py:152-220) on the
global batch; samples/s = global batch / step time.  N=1 runs the
unpartitioned module (the reference's 1-device semantics); N>1 runs
the partitioned program one mesh device per GPU (torchrun), collectives over
NCCL.  Scaling is STRONG (global batch fixed).

`value` is device-timed (CUDA events, max over ranks) with every input
resident in HBM; `e2e` repeats the measurement through the Session API with
each step's batch (x, y) copied host->device from pinned memory and the loss
read back device->host inside the timed region.  `--impl reference` times the
reference's CPU evaluator (the oracle restatement, numpy) on this host.
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


def barrier(dist):
    if dist is not None:
        dist.barrier()


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def time_reference(prog, n, inputs, steps, warmup):
    """The reference evaluator (oracle restatement; numpy on host cores)."""
    from oracle import spmd_oracle as O
    if n == 1:
        fn = lambda: O.interpret(prog.dense, inputs)
    else:
        fn = lambda: O.spmd_interpret(prog.local, prog.sharding, inputs)
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), ts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
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
        inputs = synthetic_inputs(base, seed=0, scale=wl["scale"])
        steps = max(1, min(args.steps, 3))
        warm = min(args.warmup, 1)
        med, ts = time_reference(prog, n, inputs, steps, warm)
        v = batch / med
        line = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": n, "steps": steps,
                "warmup": warm, "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": dtype, "data": "synthetic", "config": config,
                "impl": "reference",
                "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cpu_threads(), "kind": "port",
                                 "sample": f"{steps} full steps of the workload through the oracle "
                                           f"restatement of the reference evaluator ("
                                           f"{'interpret' if n == 1 else 'spmd_interpret'}); numpy "
                                           f"{np.__version__}, BLAS threads = host cores"},
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
    sess.load(inputs)
    dev = sess.device
    # eager run once (validates), then capture the whole step as one CUDA graph
    sess.run()
    sess.sync()
    sess.capture()
    for _ in range(max(3, args.warmup)):
        sess.step()
    sess.sync()
    launches_per_step = sess.launch_count()

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
        # keep sampling clocks under the same load for a short while if the region was short
        ms = dev.elapsed_ms(e0, e1)
        extra = 0
        while ms * (1 + extra) < 1500 and extra < 2000:
            for _ in range(args.steps):
                sess.step()
            extra += 1
        sess.sync()
        barrier(dist)
    ms_total = max_over_ranks(dist, ms)
    ms_step = ms_total / args.steps
    value = batch / (ms_step / 1e3)

    # ---- end to end: batch H2D from pinned host memory + loss D2H, per step
    f = sess.func
    bx = sess.local_inputs(inputs)[0]
    pin = {nm: dev.pinned(bx[nm].shape) for nm in ("x", "y") if nm in bx}
    for nm, arr in pin.items():
        arr[...] = bx[nm]
    loss_pin = dev.pinned((max(1, args.steps),))
    loss_addr = sess.result_addr(0)
    h2d = sum(a.nbytes for a in pin.values())
    import ctypes
    # warm the input pipeline (staging slots, copy stream) outside the timed region
    sess.feed(pin)
    sess.step()
    sess.sync()
    barrier(dist)
    sess.sync()
    t0 = time.perf_counter()
    dev.record(e0)
    # each step's batch is copied inside the timed region; the copy of batch
    # i+1 overlaps step i (Session.feed: copy stream + staging slots)
    # every step's loss is read back to the host (async D2H into a pinned
    # slot per step); the host waits once at the end instead of every step
    sess.feed(pin)
    for i in range(args.steps):
        if i + 1 < args.steps:
            sess.feed(pin)
        sess.step()
        R.call(dev.lib.spx_memcpy_d2h, loss_pin.ctypes.data + 4 * i, loss_addr, 4, dev.stream)
    sess.sync()
    dev.record(e1)
    sess.sync()
    wall = time.perf_counter() - t0
    e2e_ms = max_over_ranks(dist, max(dev.elapsed_ms(e0, e1), wall * 1e3))
    e2e_value = batch / (e2e_ms / args.steps / 1e3)
    h2d_total = sum_over_ranks(dist, h2d)
    d2h_total = sum_over_ranks(dist, 4)
    loss = float(loss_pin[args.steps - 1])

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
                R.K_SPLIT: "gemm_operand_split"}[kind]
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
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_full_gemm_c2_n1.json")) as fh:
            cap = json.load(fh)[0]

        def _mb(v):
            x, u = v.split()
            return float(x) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        traffic = _mb(cap["dram__bytes_read.sum"]) + _mb(cap["dram__bytes_write.sum"])
        traffic_note = (f"dram read+write bytes of one {cap['kernel'].split('(')[0].replace('void ', '')} launch "
                        f"(C2 2048x4096x1024, {cap['gpu__time_duration.sum']}) from profiles/r01_ncu_full_gemm_c2_n1.json; "
                        f"algorithmic: fp16 pieces of A 8.4 MB + B 16.8 MB read, C 33.6 MB written (C stays in L2 "
                        f"for its consumer, so DRAM sees the operand reads only)")
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

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        med, ts = time_reference(prog, n, inputs, 2, 0)
        cpu = {"value": batch / med, "unit": "samples/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"2 full steps (median {med:.2f} s) of the same workload through the oracle "
                         f"restatement of the reference's dense interpreter (interp.py:117-132), numpy "
                         f"{np.__version__}, BLAS on all host cores"}

    counts = sess.ex.comp.counts
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": n, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": config, "roofline": roofline, "streaming_roofline": streaming, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": int(h2d_total),
                        "d2h_bytes_per_step": int(d2h_total),
                        "note": "Session.feed + Session.step: every step's batch (x, y) H2D from pinned memory (the copy of batch i+1 overlaps step i) and the "
                                "loss D2H each step (async into a pinned slot per step), one host wait at the end"},
                "gpu_launches": int(launches_per_step * args.steps),
                "launches_per_step": int(launches_per_step),
                "clocks": clk.summary(), "loss": loss, "loss_finite": bool(np.isfinite(loss)),
                "collectives_per_step": counts,
                "flops_per_device_step": sess.ex.comp.flops}
        print(json.dumps(line), flush=True)
    sess.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
