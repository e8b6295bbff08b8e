"""Step-level roofline of a (localized) training-step program, per SURVEY.md §8(d).

    T_roof = max( sum_ops max(F_op / P_tc, B_op / BW_hbm),  B_nvl / BW_nvl )
    roofline.frac = T_roof / T_measured

* F_op: the reference simulator's FLOP convention (`_flops`, sim.py:86-100):
  matmul 2mkn, add/mul/neg/exp one per result element, reduce one per input
  element, everything else 0.
* P_tc: fp32 matmuls run on the tensor cores as block-scaled 3xFP16
  (three kind::f16 MMAs per fp32 FLOP), so their ceiling is the
  measured dense bf16/f16 rate / 3; elementwise and reduce FLOPs are charged
  at the fp32 CUDA-core rate (they never bind: bytes do).
* B_op: per matmul / add / mul / neg / exp / reduce, the bytes of the data its
  operands read plus its result, 4 B per element (f32/i32, ir.py:14);
  constants are immediates (0 B), views read their source (a broadcast
  operand costs its source's bytes, a transpose/reshape/tag the same bytes as
  its source), an all_slice its chunk.  Ops whose operands are all constants
  are folded at build time (0).  This is the unfused per-op minimum: a fused
  plan can beat it (it is a ceiling for the reference's op-by-op schedule).
* B_nvl: per device, sum of the ring-schedule bytes of the program's counted
  collectives (`collective_bytes`, sim.py:114-123); BW_nvl = 900 GB/s per
  direction (NVLink 5 through NVSwitch, spec -- no measured figure exists in
  MEASURED_PEAKS.json).
"""
from __future__ import annotations

COLL = ("all_gather", "all_reduce", "reduce_scatter", "all_to_all")
VIEW = ("transpose", "reshape", "tag", "broadcast")
COMPUTE = ("matmul", "add", "mul", "neg", "exp", "reduce")
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12     # B200 fp32 FMA lanes x 2 x max clock
NVLINK_GBS = 900.0


def _prod(xs):
    n = 1
    for x in xs:
        n *= int(x)
    return n


def _axes_n(op, mesh):
    axes = op.attrs["axes"] if op.kind in ("all_reduce", "reduce_scatter", "all_to_all") else \
        [a for lst in op.attrs["axes_per_dim"] for a in lst]
    return _prod(mesh.size(a) for a in axes)


def step_roofline(module, *, bf16_tflops: float, hbm_gbs: float, func: str = "main",
                  mma_per_flop: int = 3, nvlink_gbs: float = NVLINK_GBS, with_collectives: bool = True) -> dict:
    """Per-device T_roof of one step of `module` (seconds) and its parts."""
    f = module.func(func)
    mesh = getattr(module, "mesh", None)
    dims = {n: tuple(t.dims) for n, t in f.args}
    const = set()                 # values derived from constants only
    data = {n: 4 * _prod(d) for n, d in dims.items()}   # bytes of the data a value reads
    p_mm = bf16_tflops * 1e12 / mma_per_flop
    p_simt = FP32_SIMT_TFLOPS * 1e12
    bw = hbm_gbs * 1e9
    t_gemm = t_stream = 0.0
    flops = bytes_ = b_nvl = 0.0
    for op in f.ops:
        for r, t in zip(op.results, op.result_types):
            dims[r] = tuple(t.dims)
        r = op.results[0] if op.results else None
        out_b = 4 * _prod(dims[r]) if r is not None else 0
        k = op.kind
        if k == "constant":
            const.add(r)
            data[r] = 0
            continue
        ins = list(op.operands)
        if k in VIEW or k == "all_slice":
            src = ins[0]
            if src in const:
                const.add(r)
                data[r] = 0
            elif k == "all_slice":
                data[r] = out_b
            else:
                data[r] = data[src]
            continue
        if k in COLL:
            data[r] = out_b
            if with_collectives and mesh is not None:
                n = _axes_n(op, mesh)
                ob = 4 * _prod(dims[ins[0]])
                if k == "all_gather":
                    b_nvl += (n - 1) / n * out_b
                elif k == "all_reduce":
                    b_nvl += 2.0 * (n - 1) / n * ob
                else:
                    b_nvl += (n - 1) / n * ob
            continue
        if k not in COMPUTE:
            data[r] = out_b
            continue
        if all(o in const for o in ins):
            const.add(r)
            data[r] = 0
            continue
        data[r] = out_b
        b = out_b + sum(data[o] for o in ins if o not in const)
        if k == "matmul":
            m, kk = dims[ins[0]]
            fl = 2.0 * m * kk * dims[ins[1]][1]
            t_gemm += max(fl / p_mm, b / bw)
        else:
            fl = float(_prod(dims[ins[0]])) if k == "reduce" else float(_prod(dims[r]))
            t_stream += max(fl / p_simt, b / bw)
        flops += fl
        bytes_ += b
    t_compute = t_gemm + t_stream
    t_nvl = b_nvl / (nvlink_gbs * 1e9)
    return {"t_roof_s": max(t_compute, t_nvl), "t_compute_s": t_compute, "t_gemm_s": t_gemm,
            "t_stream_s": t_stream, "t_nvlink_s": t_nvl, "flops": flops, "hbm_bytes": bytes_,
            "nvlink_bytes": b_nvl, "bound": "nvlink" if t_nvl > t_compute else "compute"}
