// Fused elementwise expression kernel: the numpy per-op semantics of
// interp.py:39-67 (constant, add, mul, neg, exp, transpose/broadcast/reshape/
// tag/all_slice as strided views) evaluated as ONE HBM pass per fused group.
//
// The expression is a tiny SSA program (spx_insn) that is uniform across the
// grid; each thread evaluates it for 4 consecutive elements (float4 loads and
// stores when every input view is unit-stride or broadcast along the innermost
// dim) or 1 element (general strided path).  Operand fetch is a `switch` over
// compile-time register slots so the register file of the program stays in
// registers; the branch is warp-uniform.
#include "common.cuh"

namespace {

template <int W>
struct Vec {
  float v[W];
};

template <int W, int P>
struct Regs {
  Vec<W> in[SPX_MAX_IN];
  Vec<W> t[P];
};

#define SPX_CASE_IN(j) \
  case j:              \
    return R.in[j];
#define SPX_CASE_T(i)   \
  case SPX_REG_T + i:   \
    if (i < P) return R.t[i < P ? i : 0]; \
    break;

template <int W, int P>
SPX_DEV Vec<W> fetch(int r, const Regs<W, P>& R) {
  switch (r) {
    SPX_CASE_IN(0) SPX_CASE_IN(1) SPX_CASE_IN(2) SPX_CASE_IN(3)
    SPX_CASE_IN(4) SPX_CASE_IN(5) SPX_CASE_IN(6) SPX_CASE_IN(7)
    SPX_CASE_T(0) SPX_CASE_T(1) SPX_CASE_T(2) SPX_CASE_T(3) SPX_CASE_T(4)
    SPX_CASE_T(5) SPX_CASE_T(6) SPX_CASE_T(7) SPX_CASE_T(8) SPX_CASE_T(9)
    SPX_CASE_T(10) SPX_CASE_T(11) SPX_CASE_T(12) SPX_CASE_T(13) SPX_CASE_T(14)
    SPX_CASE_T(15) SPX_CASE_T(16) SPX_CASE_T(17) SPX_CASE_T(18) SPX_CASE_T(19)
    SPX_CASE_T(20) SPX_CASE_T(21) SPX_CASE_T(22) SPX_CASE_T(23) SPX_CASE_T(24)
    SPX_CASE_T(25) SPX_CASE_T(26) SPX_CASE_T(27)
  }
  Vec<W> z;
#pragma unroll
  for (int k = 0; k < W; ++k) z.v[k] = 0.f;
  return z;
}

// Evaluate the program; all instructions are unrolled so t[i] has a static slot.
template <int W, int P>
SPX_DEV void run_prog(const spx_ew_params& p, Regs<W, P>& R) {
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (i >= p.n_prog) break;
    const spx_insn ins = p.prog[i];
    const float imm = p.imm[i];
    Vec<W> a = fetch<W, P>(ins.a, R);
    Vec<W> b = fetch<W, P>(ins.b, R);
#pragma unroll
    for (int k = 0; k < W; ++k) R.t[i].v[k] = apply_op(ins.op, a.v[k], b.v[k], imm);
  }
}

template <int W, int P>
SPX_DEV Vec<W> result(int reg, const Regs<W, P>& R) { return fetch<W, P>(reg, R); }

// Multi-index of element e (row-major over p.dims) -> per-input offsets.
SPX_DEV void offsets(const spx_ew_params& p, int64_t e, int64_t* off) {
#pragma unroll
  for (int j = 0; j < SPX_MAX_IN; ++j)
    if (j < p.n_in) off[j] = p.in[j].off;
  int64_t rem = e;
#pragma unroll
  for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
    if (k >= p.rank) continue;
    const int64_t dk = p.dims[k];
    const int64_t ik = (k == 0) ? rem : rem % dk;
    rem = (k == 0) ? 0 : rem / dk;
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j)
      if (j < p.n_in) off[j] += ik * p.in[j].stride[k];
  }
}

// Fast 32-bit variant for rank <= 2 (the common collapsed case).
template <int W, int P>
__global__ void __launch_bounds__(256) ew_kernel(const __grid_constant__ spx_ew_params p) {
  const int d = blockIdx.y;
  const uint64_t dbase = p.base + (uint64_t)((int64_t)d * p.dev_stride);
  const float* __restrict__ fb = reinterpret_cast<const float*>(dbase);
  float* __restrict__ ob = reinterpret_cast<float*>(dbase);
  const int64_t nvec = p.numel / W;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = v * W;
    int64_t off[SPX_MAX_IN];
    if (p.rank == 1) {
#pragma unroll
      for (int j = 0; j < SPX_MAX_IN; ++j)
        if (j < p.n_in) off[j] = p.in[j].off + e * p.in[j].stride[0];
    } else if (p.rank == 2) {
      const int64_t c = e % p.dims[1], r = e / p.dims[1];
#pragma unroll
      for (int j = 0; j < SPX_MAX_IN; ++j)
        if (j < p.n_in) off[j] = p.in[j].off + r * p.in[j].stride[0] + c * p.in[j].stride[1];
    } else {
      offsets(p, e, off);
    }
    Regs<W, P> R;
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j) {
      if (j >= p.n_in) break;
      if (W == 4) {
        const int64_t sinner = p.in[j].stride[p.rank - 1];
        if (sinner == 1) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(fb + off[j]));
          R.in[j].v[0] = x.x; R.in[j].v[1 % W] = x.y; R.in[j].v[2 % W] = x.z; R.in[j].v[3 % W] = x.w;
        } else {
          const float x = __ldg(fb + off[j]);
#pragma unroll
          for (int k = 0; k < W; ++k) R.in[j].v[k] = x;
        }
      } else {
        R.in[j].v[0] = __ldg(fb + off[j]);
      }
    }
    run_prog<W, P>(p, R);
#pragma unroll
    for (int o = 0; o < SPX_MAX_OUT; ++o) {
      if (o >= p.n_out) break;
      const Vec<W> y = result<W, P>(p.out_reg[o], R);
      float* dst = ob + p.out_off[o] + e;
      if (W == 4) {
        *reinterpret_cast<float4*>(dst) = make_float4(y.v[0], y.v[1 % W], y.v[2 % W], y.v[3 % W]);
      } else {
        *dst = y.v[0];
      }
    }
  }
}

}  // namespace

int spx_launch_ew(const spx_ew_params& p, cudaStream_t s, int* nlaunch) {
  if (p.numel <= 0 || p.ndev <= 0) return 0;
  const int W = p.vec ? 4 : 1;
  if (W == 4 && (p.numel % 4 != 0)) return spx_set_error("ew: vec path needs numel %% 4 == 0");
  const int64_t nvec = p.numel / W;
  const int threads = 256;
  int64_t blocks = (nvec + threads - 1) / threads;
  const int64_t cap = (int64_t)spx_num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  dim3 grid((unsigned)blocks, (unsigned)p.ndev);
  if (p.n_prog <= 8) {
    if (W == 4) ew_kernel<4, 8><<<grid, threads, 0, s>>>(p);
    else ew_kernel<1, 8><<<grid, threads, 0, s>>>(p);
  } else {
    if (W == 4) ew_kernel<4, SPX_MAX_PROG><<<grid, threads, 0, s>>>(p);
    else ew_kernel<1, SPX_MAX_PROG><<<grid, threads, 0, s>>>(p);
  }
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}
