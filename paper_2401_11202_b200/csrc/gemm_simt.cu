// fp32 SIMT GEMM for shapes the tcgen05 path does not take (tiny or
// TMA-misaligned operands, e.g. the reference's toy 4x8 @ 8x2 programs).
// C[M,N] = A[M,K] @ B[K,N] (interp.py:43-44) with either operand possibly a
// transposed view (interp.py:51-52), batched over co-located mesh devices.
// 64x64 output tile, 16-deep K slab staged in shared memory, 4x4 per thread.
#include "common.cuh"

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256) sgemm_kernel(const __grid_constant__ spx_gemm_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.z;
  const float* A = dev_ptr(p.base, p.dev_stride, d, p.a_off);
  const float* B = dev_ptr(p.base, p.dev_stride, d, p.b_off);
  float* C = dev_ptr(p.base, p.dev_stride, d, p.c_off);
  // element strides of the logical A[m][k], B[k][n]
  const int64_t sam = p.a_mn_major ? 1 : p.lda, sak = p.a_mn_major ? p.lda : 1;
  const int64_t sbk = p.b_k_major ? 1 : p.ldb, sbn = p.b_k_major ? p.ldb : 1;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < p.K; k0 += BK) {
    for (int i = tid; i < BM * BK; i += 256) {
      int mm, kk;
      if (p.a_mn_major) { mm = i % BM; kk = i / BM; } else { kk = i % BK; mm = i / BK; }
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < p.M && gk < p.K) ? A[gm * sam + gk * sak] : 0.f;
    }
    for (int i = tid; i < BN * BK; i += 256) {
      int nn, kk;
      if (p.b_k_major) { kk = i % BK; nn = i / BK; } else { nn = i % BN; kk = i / BN; }
      const int gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < p.N && gk < p.K) ? B[gk * sbk + gn * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn < p.N) C[(int64_t)gm * p.ldc + gn] = acc[i][j];
    }
  }
}

}  // namespace

int spx_launch_gemm_simt(const spx_gemm_params& p, cudaStream_t s, int* nlaunch) {
  if (p.M <= 0 || p.N <= 0) return 0;
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, p.ndev);
  spx_launch(sgemm_kernel, grid, 256, 0, s, p);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}
