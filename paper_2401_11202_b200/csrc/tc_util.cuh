// Device helpers shared by the tcgen05 GEMM kernels (gemm_tc.cu, gemm_h3.cu):
// mbarriers, elect, TMA loads, UMMA shared-memory descriptors, MMA commits,
// TMEM loads, and the driver's tensor-map encoder.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"

namespace {

SPX_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// One lane of a converged warp (elect.sync).  The whole warp runs the issue
// loops with warp-uniform operands, so ptxas keeps descriptors in uniform
// registers; issuing from `if (lane == 0)` instead made it wrap every
// tcgen05.mma in a waterfall loop (R2UR / ELECT / VOTEU per instruction).
SPX_DEV bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(p));
  return p != 0;
}

SPX_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
SPX_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
SPX_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <bool CLUSTER>
SPX_DEV bool mbar_try(uint32_t a, uint32_t parity) {
  uint32_t done;
  if (CLUSTER) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
  return done != 0;
}
// Bounded wait: a protocol bug traps (the error surfaces to the host) instead
// of hanging the GPU.  The bound check sits behind a first try_wait so the fast path (the
// phase already complete, or completing within one hardware-suspended
// try_wait) is two instructions in the issuing warp's loop.
template <bool CLUSTER>
SPX_DEV void mbar_wait_slow(uint32_t a, uint32_t parity) {
  const long long t0 = clock64();
  for (int it = 1;; ++it) {
    if (mbar_try<CLUSTER>(a, parity)) return;
    if ((it & 1023) == 0 && clock64() - t0 > 20000000000LL) __trap();
  }
}
// CLUSTER = acquire at cluster scope (peer arrivals).
template <bool CLUSTER = false>
SPX_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (!mbar_try<CLUSTER>(a, parity)) mbar_wait_slow<CLUSTER>(a, parity);
}

SPX_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor (sm_100 version 1).  Layout type 2 =
// SWIZZLE_128B (16B atoms; K-major operands), 1 = SWIZZLE_128B_BASE32B (32B
// atoms; MN-major tf32 operands).
SPX_DEV uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

// MMA completion -> barrier (CG=2: the barrier at the same offset in both CTAs).
template <int CG>
SPX_DEV void mma_commit(uint64_t* bar) {
  if (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
  }
}

SPX_DEV void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D fp32 map {inner, outer, device}; box {32, box_outer, 1}; 128B swizzle
// with 16B atoms (K-major operands) or 32B atoms (MN-major operands).
int make_map(CUtensorMap* map, uint64_t addr, uint64_t inner, uint64_t outer, uint64_t ndev, uint64_t row_bytes,
             uint64_t dev_bytes, uint32_t box_outer, bool mn_major) {
  auto enc = get_encode();
  if (!enc) return spx_set_error("cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {inner, outer, ndev};
  cuuint64_t strides[2] = {row_bytes, dev_bytes ? dev_bytes : row_bytes * outer};
  cuuint32_t box[3] = {32, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, reinterpret_cast<void*>(addr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return spx_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

}  // namespace
