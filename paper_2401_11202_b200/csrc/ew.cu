// Fused elementwise expression kernel: the numpy per-op semantics of
// interp.py:39-67 (constant, add, mul, neg, exp, transpose/broadcast/reshape/
// tag/all_slice as strided views) evaluated as ONE HBM pass per fused group.
//
// Vector path (views collapsed to rank <= 2 with innermost stride 0 or 1 and
// 16B alignment): one float4 granule per thread per iteration, grid-stride,
// all NIN loads issued before the program runs.  General path: any rank <= 6,
// arbitrary strides, one element per thread.
#include "interp.cuh"

namespace {

template <int NIN>
__global__ void __launch_bounds__(256) ew_vec_kernel(const __grid_constant__ spx_ew_params p) {
  const int d = blockIdx.y;
  const float* __restrict__ fb = dev_ptr(p.base, p.dev_stride, d, 0);
  float* __restrict__ ob = dev_ptr(p.base, p.dev_stride, d, 0);
  const int64_t nvec = p.numel >> 2;
  const bool two_d = p.rank == 2;
  const int64_t cols = two_d ? p.dims[1] : p.numel;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += step) {
    const int64_t e = v << 2;
    int64_t r = 0, c = e;
    if (two_d) {
      r = e / cols;
      c = e - r * cols;
    }
    RegFile<4> f;
#pragma unroll
    for (int j = 0; j < NIN; ++j) {
      if (j >= p.n_in) break;
      const int64_t s1 = p.in[j].stride[p.rank - 1];
      const int64_t off = p.in[j].off + (two_d ? r * p.in[j].stride[0] : 0) + (s1 ? c : 0);
      if (s1) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(fb + off));
        f.r[j].v[0] = x.x; f.r[j].v[1] = x.y; f.r[j].v[2] = x.z; f.r[j].v[3] = x.w;
      } else {
        const float x = __ldg(fb + off);
        f.r[j].v[0] = x; f.r[j].v[1] = x; f.r[j].v[2] = x; f.r[j].v[3] = x;
      }
    }
    run_program<4>(p.prog, p.imm, p.n_prog, f);
#pragma unroll
    for (int o = 0; o < SPX_MAX_OUT; ++o) {
      if (o >= p.n_out) break;
      const Vec<4> y = f.get(p.out_reg[o]);
      *reinterpret_cast<float4*>(ob + p.out_off[o] + e) = make_float4(y.v[0], y.v[1], y.v[2], y.v[3]);
    }
  }
}

__global__ void __launch_bounds__(256) ew_gen_kernel(const __grid_constant__ spx_ew_params p) {
  const int d = blockIdx.y;
  const float* __restrict__ fb = dev_ptr(p.base, p.dev_stride, d, 0);
  float* __restrict__ ob = dev_ptr(p.base, p.dev_stride, d, 0);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.numel;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t off[SPX_MAX_IN];
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j) off[j] = p.in[j].off;
    int64_t rem = e;
#pragma unroll
    for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
      if (k >= p.rank) continue;
      const int64_t ik = (k == 0) ? rem : rem % p.dims[k];
      rem = (k == 0) ? 0 : rem / p.dims[k];
#pragma unroll
      for (int j = 0; j < SPX_MAX_IN; ++j) off[j] += ik * p.in[j].stride[k];
    }
    RegFile<1> f;
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j) {
      if (j >= p.n_in) break;
      f.r[j].v[0] = __ldg(fb + off[j]);
    }
    run_program<1>(p.prog, p.imm, p.n_prog, f);
#pragma unroll
    for (int o = 0; o < SPX_MAX_OUT; ++o) {
      if (o >= p.n_out) break;
      ob[p.out_off[o] + e] = f.get(p.out_reg[o]).v[0];
    }
  }
}

unsigned blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)spx_num_sms() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

int spx_launch_ew(const spx_ew_params& p, cudaStream_t s, int* nlaunch) {
  if (p.numel <= 0 || p.ndev <= 0) return 0;
  if (p.n_prog > SPX_MAX_PROG || p.n_in > SPX_MAX_IN || p.n_out > SPX_MAX_OUT)
    return spx_set_error("ew: program exceeds ABI limits");
  const bool vec = p.vec && p.numel % 4 == 0 && p.rank <= 2;
  if (vec) {
    dim3 grid(blocks_for(p.numel / 4), (unsigned)p.ndev);
    switch (p.n_in) {
      case 0:
      case 1: ew_vec_kernel<1><<<grid, 256, 0, s>>>(p); break;
      case 2: ew_vec_kernel<2><<<grid, 256, 0, s>>>(p); break;
      case 3: ew_vec_kernel<3><<<grid, 256, 0, s>>>(p); break;
      case 4: ew_vec_kernel<4><<<grid, 256, 0, s>>>(p); break;
      default: ew_vec_kernel<SPX_MAX_IN><<<grid, 256, 0, s>>>(p);
    }
  } else {
    ew_gen_kernel<<<dim3(blocks_for(p.numel), (unsigned)p.ndev), 256, 0, s>>>(p);
  }
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}
