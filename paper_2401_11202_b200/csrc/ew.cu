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

// U float4 granules per thread per iteration (loads hoisted).  Index math is
// 32-bit relative to per-input base pointers (numel < 2^31).  This generic
// interpreter is the fallback; the model zoo's programs run as the
// compile-time-specialised kernels of ew_static.cu.
template <int NIN, int U>
__global__ void __launch_bounds__(256) ew_vec_kernel(const __grid_constant__ spx_ew_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const float* __restrict__ fb = dev_ptr(p.base, p.dev_stride, d, 0);
  float* __restrict__ ob = dev_ptr(p.base, p.dev_stride, d, 0);
  const uint32_t nvec = (uint32_t)(p.numel >> 2);
  const int rk = p.rank;
  const uint32_t cols = (uint32_t)p.dims[rk - 1];     // innermost extent (float4 along it)
  const uint32_t step = gridDim.x * blockDim.x;
  const float* in_base[NIN];
  bool s1[NIN];
#pragma unroll
  for (int j = 0; j < NIN; ++j) {
    in_base[j] = fb + p.in[j].off;
    s1[j] = p.in[j].stride[rk - 1] != 0;
  }
  for (uint32_t v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < nvec; v0 += step * U) {
    Vec<4> x[U][NIN];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t v = v0 + u * step;
      if (v >= nvec) break;
      const uint32_t e = v << 2;
      uint32_t q = rk > 1 ? e / cols : 0u;            // index over the outer dims
      const uint32_t c = e - q * cols;
      int64_t outer[NIN];
#pragma unroll
      for (int j = 0; j < NIN; ++j) outer[j] = 0;
#pragma unroll
      for (int k = SPX_MAX_RANK - 2; k >= 0; --k) {   // decompose q over dims[0 .. rk-2]
        if (k > rk - 2) continue;
        const uint32_t dk = (uint32_t)p.dims[k];
        const uint32_t ik = k == 0 ? q : q % dk;
        q = k == 0 ? 0u : q / dk;
#pragma unroll
        for (int j = 0; j < NIN; ++j) outer[j] += (int64_t)ik * p.in[j].stride[k];
      }
#pragma unroll
      for (int j = 0; j < NIN; ++j) {
        if (j >= p.n_in) break;
        const float* src = in_base[j] + outer[j];
        if (s1[j]) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(src + c));
          x[u][j].v[0] = t.x; x[u][j].v[1] = t.y; x[u][j].v[2] = t.z; x[u][j].v[3] = t.w;
        } else {
          const float t = __ldg(src);
          x[u][j].v[0] = t; x[u][j].v[1] = t; x[u][j].v[2] = t; x[u][j].v[3] = t;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t v = v0 + u * step;
      if (v >= nvec) break;
      RegFile<4> f;
#pragma unroll
      for (int j = 0; j < NIN; ++j) f.r[j] = x[u][j];
      run_program<4>(p.prog, p.imm, p.n_prog, f);
#pragma unroll
      for (int o = 0; o < SPX_MAX_OUT; ++o) {
        if (o >= p.n_out) break;
        const Vec<4> y = f.get(p.out_reg[o]);
        *reinterpret_cast<float4*>(ob + p.out_off[o] + ((size_t)v << 2)) =
            make_float4(y.v[0], y.v[1], y.v[2], y.v[3]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) ew_gen_kernel(const __grid_constant__ spx_ew_params p) {
  SPX_PDL_ENTRY();
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
  const bool vec = p.vec && p.numel % 4 == 0 && p.numel < (int64_t(1) << 31);
  if (vec) {
    const int64_t nv = p.numel / 4;
    auto grid_u = [&](int u) { return dim3(blocks_for((nv + u - 1) / u), (unsigned)p.ndev); };
    switch (p.n_in) {
      case 0:
      case 1: spx_launch(ew_vec_kernel<1, 1>, grid_u(1), 256, 0, s, p); break;
      case 2: spx_launch(ew_vec_kernel<2, 1>, grid_u(1), 256, 0, s, p); break;
      case 3: spx_launch(ew_vec_kernel<3, 1>, grid_u(1), 256, 0, s, p); break;
      case 4: spx_launch(ew_vec_kernel<4, 1>, grid_u(1), 256, 0, s, p); break;
      default: spx_launch(ew_vec_kernel<SPX_MAX_IN, 1>, grid_u(1), 256, 0, s, p);
    }
  } else {
    spx_launch(ew_gen_kernel, dim3(blocks_for(p.numel), (unsigned)p.ndev), 256, 0, s, p);
  }
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}
