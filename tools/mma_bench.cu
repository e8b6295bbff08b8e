// tcgen05.mma kind::tf32 issue-rate microbenchmark (development tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_bench tools/mma_bench.cu -lcuda
// One CTA per SM; one elected thread issues ITERS x 12 MMAs (the 3xTF32
// k-block pattern) into TMEM accumulators from garbage operands and commits;
// reports achieved tf32 TFLOP/s for each variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         ((uint64_t)2 << 61);
}

// VAR: 0 = A in TMEM, one accumulator; 1 = A in TMEM, hi.hi and corrections in two
// accumulators; 2 = A in smem (SS), one accumulator
template <int N, int VAR>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint64_t db = sdesc(smem_u32(sm)), db2 = sdesc(smem_u32(sm + 32768));
    const uint64_t da = sdesc(smem_u32(sm + 65536)), da2 = sdesc(smem_u32(sm + 98304));
    const uint32_t acc0 = tm, acc1 = tm + N;
    const uint32_t ahi = tm + 384, alo = tm + 416;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (VAR == 2) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc0),
                       "l"(da + kk * 2), "l"(db2 + kk * 2), "r"(idesc), "r"(1));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc0),
                       "l"(da2 + kk * 2), "l"(db + kk * 2), "r"(idesc), "r"(1));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc0),
                       "l"(da + kk * 2), "l"(db + kk * 2), "r"(idesc), "r"(1));
        } else {
          const uint32_t c1 = VAR == 1 ? acc1 : acc0;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(c1),
                       "r"(ahi + kk * 8), "l"(db2 + kk * 2), "r"(idesc), "r"(1));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(c1),
                       "r"(alo + kk * 8), "l"(db + kk * 2), "r"(idesc), "r"(1));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(acc0),
                       "r"(ahi + kk * 8), "l"(db + kk * 2), "r"(idesc), "r"(1));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    }
    if (blockIdx.x == 0) *cycles = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

template <int N, int VAR>
void run(const char* name) {
  const int iters = 20000, smem = 131072 + 1024;
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  cudaFuncSetAttribute(bench<N, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<N, VAR><<<148, 128, smem>>>(10, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<N, VAR><<<148, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 8 * 12.0 * iters * 148;
  printf("%-34s N=%3d  %8.3f ms  %7.1f TF/s tf32  %6.1f cyc/MMA  %s\n", name, N, ms, flops / ms / 1e9,
         (double)c / (iters * 12.0), cudaGetErrorString(err));
  cudaFree(cyc);
}

int main() {
  run<128, 0>("A-TMEM one accumulator");
  run<128, 1>("A-TMEM two accumulators");
  run<128, 2>("A-SMEM one accumulator");
  run<256, 0>("A-TMEM one accumulator");
  run<256, 2>("A-SMEM one accumulator");
  run<64, 0>("A-TMEM one accumulator");
  return 0;
}
