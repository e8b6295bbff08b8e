// Block-scaled fp16 pieces for the 3xFP16 GEMM (gemm_h3.cu): the per-block
// scale choice and the hi/lo conversion, shared by the standalone split kernel
// and the elementwise kernels that emit pieces of their output (ew_static.cu).
#pragma once
#include <cuda_fp16.h>
#include "common.cuh"

constexpr int H3_BLOCK = 128;                 // scale block edge
constexpr int H3_CL = 4;                      // CTAs per block (cluster), 32 rows each
constexpr int H3_ROWS = H3_BLOCK / H3_CL;
constexpr int H3_V = H3_ROWS * (H3_BLOCK / 4) / 256;   // float4 per thread at 256 threads (4)

// Power-of-two exponent e with max * 2^e in [2^14, 2^15), clamped to +-60
// (zero / inf / NaN blocks: e = 0).
SPX_DEV int h3_scale_exp(float m) {
  const int E = (int)((__float_as_uint(m) >> 23) & 0xFF);
  int e = (m == 0.f || E == 255) ? 0 : 141 - E;
  return e < -60 ? -60 : (e > 60 ? 60 : e);
}
SPX_DEV float h3_pow2(int e) { return __uint_as_float((uint32_t)(127 + e) << 23); }

// Would the block's scale have been clamped (finite, nonzero max outside
// [2^-45, 2^75]: its small elements lose precision in the fp16 pieces)?
// Counted so the host can report it instead of degrading silently.
SPX_DEV bool h3_out_of_range(float m) {
  const int E = (int)((__float_as_uint(m) >> 23) & 0xFF);
  if (m == 0.f || E == 255) return false;
  const int e = 141 - E;
  return e < -60 || e > 60;
}

SPX_DEV float h3_absmax4(float m, float4 x) {
  return fmaxf(m, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
}

// Split form of h3_cluster_max: `arrive` publishes this CTA's partial maximum
// to every CTA of the cluster and arrives on the cluster barrier (release);
// `wait` completes the barrier (acquire) and returns the block maximum.  Work
// issued between the two -- the elementwise kernel's fp32 output stores, the
// next block's loads -- is not waited for by the release.
SPX_DEV void h3_cluster_max_arrive(float m, float* wmax, float* cmax, int crank) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) wmax[warp] = m;
  __syncthreads();
  if (tid < H3_CL) {
    float mm = wmax[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) mm = fmaxf(mm, wmax[w]);
    uint32_t dst;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(dst)
                 : "r"((uint32_t)__cvta_generic_to_shared(&cmax[crank])), "r"(tid));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst), "f"(mm) : "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
SPX_DEV float h3_cluster_max_wait(const float* cmax) {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  float r = cmax[0];
#pragma unroll
  for (int w = 1; w < H3_CL; ++w) r = fmaxf(r, cmax[w]);
  return r;
}

// Maximum over the H3_CL CTAs of a cluster (each holding its partial max `m`
// per thread); every thread of every CTA returns the block maximum.
// wmax: __shared__ float[8], cmax: __shared__ float[H3_CL].
SPX_DEV float h3_cluster_max(float m, float* wmax, float* cmax, int crank) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) wmax[warp] = m;
  __syncthreads();
  if (tid < H3_CL) {
    float mm = wmax[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) mm = fmaxf(mm, wmax[w]);
    uint32_t dst;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(dst)
                 : "r"((uint32_t)__cvta_generic_to_shared(&cmax[crank])), "r"(tid));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst), "f"(mm) : "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  float r = cmax[0];
#pragma unroll
  for (int w = 1; w < H3_CL; ++w) r = fmaxf(r, cmax[w]);
  return r;
}

// hi = rn(x * up), lo = rn(x * up - hi) for 4 consecutive elements at o
// (n < 4: only the first n exist).
SPX_DEV void h3_store4(__half* hi, __half* lo, int64_t o, float4 v, float up, int n) {
  const float y0 = __fmul_rn(v.x, up), y1 = __fmul_rn(v.y, up);
  const float y2 = __fmul_rn(v.z, up), y3 = __fmul_rn(v.w, up);
  const __half2 h01 = __floats2half2_rn(y0, y1), h23 = __floats2half2_rn(y2, y3);
  const float2 b01 = __half22float2(h01), b23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn(__fsub_rn(y0, b01.x), __fsub_rn(y1, b01.y));
  const __half2 l23 = __floats2half2_rn(__fsub_rn(y2, b23.x), __fsub_rn(y3, b23.y));
  if (n >= 4) {
    uint2 hv, lv;
    hv.x = *reinterpret_cast<const uint32_t*>(&h01); hv.y = *reinterpret_cast<const uint32_t*>(&h23);
    lv.x = *reinterpret_cast<const uint32_t*>(&l01); lv.y = *reinterpret_cast<const uint32_t*>(&l23);
    *reinterpret_cast<uint2*>(hi + o) = hv;
    *reinterpret_cast<uint2*>(lo + o) = lv;
  } else {
    const __half hh[4] = {__low2half(h01), __high2half(h01), __low2half(h23), __high2half(h23)};
    const __half ll[4] = {__low2half(l01), __high2half(l01), __low2half(l23), __high2half(l23)};
    for (int j = 0; j < n; ++j) {
      hi[o + j] = hh[j];
      lo[o + j] = ll[j];
    }
  }
}
