// Block-scaled 3xFP16 tcgen05 GEMM for the reference's fp32 `matmul`
// (interp.py:43-44: numpy `@` on float32 arrays).
//
// The tf32 kernel (gemm_tc.cu) needs three kind::tf32 MMAs per fp32 product
// and splits the operands on the SM.  kind::f16 runs at twice the tf32 rate,
// so three fp16 MMAs cost half as much -- if fp16 pieces can carry fp32
// precision.  They can, with a power-of-two scale per 128 x 128 block:
//
//   split:  s = 2^e with max|x| * s in [2^14, 2^15) over the block,
//           hi = fp16_rn(x * s), lo = fp16_rn(x * s - hi)      (x * s - hi exact)
//           => x * s = hi + lo + r, |r| <= 2^-22 |x * s| (or 2^-25 absolute,
//              i.e. 2^-40 of the block maximum, where lo is subnormal)
//   GEMM:   per 128-wide k chunk, D_c = hi.lo + hi.hi + lo.hi (tensor core,
//           products exact in fp32), folded into fp32 registers as
//           acc += D_c * (1 / (s_A(block) * s_B(block)))      (exact power of 2)
//
// 128 x 128 blocks are symmetric in rows and columns, so the same pieces serve
// a tensor used K-major or MN-major, and one scale per (CTA tile, k chunk) is
// all the drain needs: an A chunk of a CTA is one block of A's rows, a B chunk
// of a pair tile one block of B's columns.  Per-chunk fp32 promotion also keeps
// the tensor core's truncating accumulation out of the error (see gemm_tc.cu).
// Error vs float64: ~1e-6 max-normalised at any K (fp32 parity bar 1e-5,
// SPEC.md:92).  Scales are clamped to 2^+-60 (blocks with max |x| outside
// [2^-45, 2^75] lose precision; fp32 data of a training step is far inside).
//
// Two kernels per GEMM, both HBM- or tensor-bound and PDL-chained:
//   split_h16_kernel  one CTA per 128 x 128 block of an fp32 operand view:
//                     read 4 B, write hi + lo (4 B) per element, one scale;
//   gemm_h3_kernel    persistent, CTA pairs (cta_group::2, 256 x 128 tiles,
//                     each CTA holds 128 A rows and 64 B columns), pure TMA ->
//                     MMA -> drain: warp 0 TMA (both CTAs' loads complete on
//                     the leader's barrier), warp 1 of the leader issues
//                     kind::f16 MMAs (A collector reused by hi.lo / hi.hi),
//                     warps 4-7 fold TMEM chunks with their scale and store C
//                     through TMA.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cuda_fp16.h>
#include "common.cuh"
#include "tc_util.cuh"
#include "h3_split.cuh"

namespace {

constexpr int HB = 128;                  // scale block edge = A rows per CTA = K per chunk
constexpr int HBK = 64;                  // fp16 per 128-byte swizzle row = K per k-block
constexpr int H_CG = 2;
constexpr int H_A_BYTES = HB * HBK * 2;      // 16 KB per piece

struct SplitArgs {
  uint64_t src;          // device-0 address of element (0, 0) of the fp32 view
  int64_t src_dev;       // bytes between devices
  int64_t ld;            // row pitch (elements)
  int rows, cols;
  uint64_t dst;          // device-0 address of the pieces [2][rows][pitch] fp16
  int64_t dst_dev;       // bytes
  int64_t pitch;         // halves (multiple of 8: 16 B TMA pitch)
  uint64_t scl;          // device-0 address of 1/s per block [rb][cb] (fp32)
  int64_t scl_dev;       // bytes
  int cb;
};

// A cluster of H3_CL CTAs splits one 128 x 128 block (CTA rank r takes rows
// 32r..32r+31): the block maximum is exchanged through distributed shared
// memory, so a 1024 x 1024 operand spreads over 256 CTAs instead of 64.
__device__ uint32_t g_h3_range_split = 0;   // blocks whose scale was clamped (h3_out_of_range)

// split_block: block (by, bx) of operand `a` on device `dev`, this CTA's quarter.
SPX_DEV void split_block(const SplitArgs& a, int bx, int by, int crank, int dev) {
  __shared__ float wmax[8];
  __shared__ float cmax[H3_CL];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = by * HB + crank * H3_ROWS, c0 = bx * HB;
  const float* src = reinterpret_cast<const float*>(a.src + (uint64_t)((int64_t)dev * a.src_dev));
  const bool vec = ((a.src | (uint64_t)a.src_dev | (uint64_t)(a.ld * 4)) & 15) == 0 && c0 + HB <= a.cols;
  float4 v[H3_V];
  float m = 0.f;
  const int c = c0 + lane * 4;
#pragma unroll
  for (int i = 0; i < H3_V; ++i) {
    const int r = r0 + i * 8 + warp;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < a.rows) {
      const float* p = src + (int64_t)r * a.ld + c;
      if (vec) {
        x = *reinterpret_cast<const float4*>(p);
      } else {
        if (c < a.cols) x.x = p[0];
        if (c + 1 < a.cols) x.y = p[1];
        if (c + 2 < a.cols) x.z = p[2];
        if (c + 3 < a.cols) x.w = p[3];
      }
    }
    v[i] = x;
    m = h3_absmax4(m, x);
  }
  m = h3_cluster_max(m, wmax, cmax, crank);
  const int e = h3_scale_exp(m);
  const float up = h3_pow2(e);
  if (threadIdx.x == 0 && crank == 0) {
    reinterpret_cast<float*>(a.scl + (uint64_t)((int64_t)dev * a.scl_dev))[by * a.cb + bx] = h3_pow2(-e);
    if (h3_out_of_range(m)) atomicAdd(&g_h3_range_split, 1u);
  }
  __half* hi = reinterpret_cast<__half*>(a.dst + (uint64_t)((int64_t)dev * a.dst_dev));
  __half* lo = hi + (int64_t)a.rows * a.pitch;
#pragma unroll
  for (int i = 0; i < H3_V; ++i) {
    const int r = r0 + i * 8 + warp;
    if (r >= a.rows || c >= a.cols) continue;
    h3_store4(hi, lo, (int64_t)r * a.pitch + c, v[i], up, min(4, a.cols - c));
  }
}

__global__ void __cluster_dims__(H3_CL, 1, 1) __launch_bounds__(256)
split_h16_kernel(const __grid_constant__ SplitArgs a) {
  SPX_PDL_ENTRY();
  split_block(a, blockIdx.x / H3_CL, blockIdx.y, blockIdx.x % H3_CL, blockIdx.z);
}

// Several independent splits in one launch (consecutive SPX_K_SPLIT records
// of a stream, e.g. the hoisted splits of every weight at the start of a
// step): one grid over all their 128 x 128 blocks, so the per-launch ramp and
// tail are paid once and the loads of one CTA overlap the stores of others.
// Cluster c belongs to the job j with start[j] <= c < start[j + 1].
constexpr int SPLIT_MAX_JOBS = 48;
struct SplitBatch {
  int n;
  int start[SPLIT_MAX_JOBS + 1];       // first cluster of each job (start[n] = total)
  SplitArgs job[SPLIT_MAX_JOBS];
};

__global__ void __cluster_dims__(H3_CL, 1, 1) __launch_bounds__(256)
split_h16_batch_kernel(const __grid_constant__ SplitBatch b) {
  const int cl = blockIdx.x / H3_CL;
  int lo = 0, hi = b.n - 1;            // last j with start[j] <= cl
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b.start[mid] <= cl) lo = mid; else hi = mid - 1;
  }
  const SplitArgs& a = b.job[lo];
  const int c = cl - b.start[lo];
  SPX_PDL_ENTRY();
  split_block(a, c % a.cb, c / a.cb, blockIdx.x % H3_CL, blockIdx.y);
}

struct H3Args {
  int M, N, K;
  int a_mn_major, b_k_major;
  int tiles_m, tiles_n, tiles;
  int group_m;                         // tile raster: groups of group_m M-tiles, M fastest inside a group
  int tma_store;
  uint64_t c_base;
  int64_t dev_stride;                  // bytes (C)
  int64_t ldc;
  uint64_t sa, sb;                     // device-0 addresses of the operand scales
  int64_t sa_dev, sb_dev;              // bytes
  int64_t sa_m, sa_k, sb_n, sb_k;      // element strides of the scale grids
  int rb_a;                            // A row blocks (guards the last pair's second CTA)
  // split-K (splits > 1): unit u = tile u / splits, k chunks [nc s / S, nc (s+1) / S);
  // every unit stores its partial 32-row slices to the workspace [S][M][N] and
  // counts them into a per-slice flag; the LAST unit of a slice to arrive folds
  // all S partials in split order (deterministic) and stores C.  No unit waits
  // for another, so units need not be co-resident.
  int splits, units;
  uint64_t flag_base;                  // uint32 [tiles][2 CTAs][BN/128][4 warps] per device, zero between launches
  int64_t flag_dev;                    // bytes
  uint64_t ws_base;                    // device-0 address of the partials
  int64_t ws_dev;                      // bytes
  // dynamic unit scheduling (dyn = 1): pairs take units from a global counter
  // (sched[0]; sched[1] counts pairs that ran dry -- the last one resets both
  // for the next launch), so pairs that become resident late (SMs held by a
  // concurrent kernel on another stream) find fewer units instead of holding
  // back a static share
  int dyn;
  uint64_t sched;                      // uint32[2], zero between launches
  int fold_tma;                        // split-K: the last unit pulls the other partials by TMA
};

template <bool LEADER_BAR>
SPX_DEV void tma_load_4d(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2, int c3) {
  if (LEADER_BAR)
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

// collector: 0 none, 1 fill A, 2 last use of A
template <int COLLECT>
SPX_DEV void mma_f16_ss(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
#define SPX_MMA16(SUFFIX)                                                                    \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                             \
               "tcgen05.mma.cta_group::2.kind::f16" SUFFIX " [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d), \
               "l"(da), "l"(db), "r"(idesc), "r"(acc))
  if (COLLECT == 1) SPX_MMA16(".collector::a::fill");
  else if (COLLECT == 2) SPX_MMA16(".collector::a::lastuse");
  else SPX_MMA16("");
#undef SPX_MMA16
}

// Tile configuration: BN output columns per CTA pair (each CTA holds BN/2 B
// columns and drains a 128 x BN accumulator with BN/128 drain warpgroups).
//   BN = 128: 48 KB stages x 4; 256 threads (WG0 TMA/MMA, WG1 drain)
//   BN = 256: 64 KB stages x 3; 384 threads (WG0, WG1-2 drain column halves),
//             the largest MMA (256 x 256 x 16): per SM the tensor core then
//             reads 52 B/cycle of operands from shared memory instead of 73
//             (+ 42 instead of 64 B/cycle of TMA writes) -- BN = 128 sits just
//             above the shared-memory port once TMA traffic is counted.
template <int BN>
struct H3Cfg {
  static constexpr int BNH = BN / H_CG;
  static constexpr int B_BYTES = BNH * HBK * 2;
  static constexpr int STAGE = 2 * H_A_BYTES + 2 * B_BYTES;
  static constexpr int RS = BN == 128 ? 4 : 3;
  static constexpr int NDG = BN / 128;                      // drain warpgroups
  static constexpr int THREADS = 128 * (1 + NDG);
  static constexpr int BAR_OFF = RS * STAGE;
  static constexpr int STG_OFF = BAR_OFF + 1024;
  static constexpr int STG_WARP = BN == 128 ? 8192 : 4096;  // 2 or 1 staging slices per drain warp
  static constexpr int TOTAL = STG_OFF + 4 * NDG * STG_WARP + 1024;
  static constexpr int TMEM_COLS = 2 * BN;
};

template <int BN>
__global__ void __launch_bounds__(H3Cfg<BN>::THREADS, 1)
gemm_h3_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
               const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ CUtensorMap tma_w,
               const __grid_constant__ H3Args args) {
  using S = H3Cfg<BN>;
  constexpr int RS = S::RS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* raw_empty = raw_full + RS;
  uint64_t* tfull = raw_empty + RS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  constexpr int UQ = 4;                       // unit queue (dynamic scheduling)
  uint64_t* uq_full = tempty + 4;             // 8 B after tmem_slot
  uint64_t* uq_empty = uq_full + UQ;
  volatile int* uq = reinterpret_cast<volatile int*>(uq_empty + UQ);
  uint64_t* fold_bar = uq_empty + UQ + 2;     // split-K fold: one barrier per drain warp (4)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (args.K + HBK - 1) / HBK;
  uint32_t crank = 0;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int pair0 = blockIdx.x / H_CG, npairs = gridDim.x / H_CG;
  auto a_hi = [&](int s) { return smem + s * S::STAGE; };
  auto b_hi = [&](int s) { return smem + s * S::STAGE + 2 * H_A_BYTES; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4 * S::NDG * H_CG);
    }
    for (int q = 0; q < UQ; ++q) {
      mbar_init(&uq_full[q], 1);
      // consumers: the leader's MMA warp and drain warps, the peer's producer and drain warps
      mbar_init(&uq_empty[q], 2 + 2 * 4 * S::NDG);
    }
    for (int q = 0; q < 4; ++q) mbar_init(&fold_bar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(S::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_d = *tmem_slot;
  SPX_PDL_ENTRY();

  const int nch = (nk + 1) / 2;               // 128-wide k chunks
  // unit -> (tile, split, first chunk, chunk count)
  auto unit_of = [&](int u, int& t, int& sp, int& c0, int& ncu) {
    t = u / args.splits;
    sp = u - t * args.splits;
    c0 = (int)(((long long)nch * sp) / args.splits);
    ncu = (int)(((long long)nch * (sp + 1)) / args.splits) - c0;
  };
  // Tile raster: groups of group_m M-tiles (row panels of A), M fastest inside
  // a group, groups in order.  The pairs working at the same time then cover a
  // ~group_m x (pairs / group_m) rectangle of tiles whose A and B panels stay in
  // L2 together (the host picks group_m ~ sqrt(pairs * BN / 256), the
  // footprint minimum); group_m = tiles_m is plain M-fastest order.
  auto tile_of = [&](int t, int& m0, int& n0, int& dev) {
    const int per_dev = args.tiles_m * args.tiles_n;
    dev = t / per_dev;
    int r = t - dev * per_dev;
    const int gsz = args.group_m * args.tiles_n;
    const int g = r / gsz;
    r -= g * gsz;
    const int mf = g * args.group_m;
    const int gm = min(args.group_m, args.tiles_m - mf);
    const int n_blk = r / gm;
    m0 = (mf + (r - n_blk * gm)) * (HB * H_CG);
    n0 = n_blk * BN;
  };

  // The j-th unit of this pair (static: pair0 + j * npairs).  Dynamic: the
  // leader's producer warp fetches it from the global counter and publishes it
  // in both CTAs' queue slot (the peer's through distributed shared memory);
  // every other consumer warp reads its own CTA's slot and releases it on the
  // leader's empty barrier.  A unit >= units ends every role's loop.
  // Claims: every pair's first unit is its static one (pair0, no atomic on the
  // critical path of small GEMMs); later units come from the counter, claimed
  // one unit AHEAD (right after publishing the current one) so the atomic's
  // latency hides behind the current unit's loads.  Unit = npairs + claim.
  int pref = 0;
  auto get_unit = [&](int j, bool fetcher) -> int {
    if (!args.dyn) return pair0 + j * npairs;
    const int slot = j & (UQ - 1);
    const uint32_t ph = (uint32_t)((j / UQ) & 1);
    int u = 0;
    if (fetcher) {
      mbar_wait<true>(&uq_empty[slot], ph ^ 1u);
      if (lane == 0) {
        uint32_t* cnt = reinterpret_cast<uint32_t*>(args.sched);
        u = j == 0 ? pair0 : pref;
        uq[slot] = u;
        uint32_t r_uq, r_full;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(r_uq) : "r"(smem_u32((const void*)&uq[slot])));
        asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(r_full) : "r"(smem_u32(&uq_full[slot])));
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(r_uq), "r"(u) : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r_full) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&uq_full[slot])) : "memory");
        if (u < args.units) {
          pref = npairs + (int)atomicAdd(cnt, 1u);          // claim the next unit now
        } else if (atomicAdd(cnt + 1, 1u) == (uint32_t)(npairs - 1)) {
          // this pair ran dry, and it is the last one: reset for the next launch
          atomicExch(cnt, 0u);
          atomicExch(cnt + 1, 0u);
        }
      }
      u = __shfl_sync(0xffffffffu, u, 0);
    } else {
      mbar_wait<true>(&uq_full[slot], ph);
      u = uq[slot];
      __syncwarp();
      if (lane == 0) {
        uint32_t r;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(&uq_empty[slot])));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
      }
    }
    return u;
  };

  if (warp < 4) {
    if (BN > 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 0) {
      // ---------------- TMA producer (both CTAs; loads land on the leader's barrier) ----------------
      uint32_t lead_full0;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead_full0) : "r"(smem_u32(&raw_full[0])));
      int g = 0;
      for (int j = 0;; ++j) {
        const int u = get_unit(j, crank == 0);
        if (u >= args.units) break;
        int t, sp, c0, ncu, m0, n0, dev;
        unit_of(u, t, sp, c0, ncu);
        tile_of(t, m0, n0, dev);
        m0 += (int)crank * HB;
        const int nb0 = n0 + (int)crank * S::BNH;
        const int kbe = min(nk, 2 * (c0 + ncu));
        for (int kb = 2 * c0; kb < kbe; ++kb, ++g) {
          const int s = g % RS;
          mbar_wait(&raw_empty[s], ((g / RS) & 1) ^ 1);
          if (elect_one()) {
            if (crank == 0) mbar_expect_tx(&raw_full[s], (uint32_t)(H_CG * S::STAGE));
            const uint32_t bar = lead_full0 + (uint32_t)(s * 8);
            const int k0 = kb * HBK;
            uint8_t* st = a_hi(s);
#pragma unroll
            for (int piece = 0; piece < 2; ++piece) {
              uint8_t* da = st + piece * H_A_BYTES;
              if (args.a_mn_major) {
                tma_load_4d<true>(da, &tma_a, bar, m0, k0, piece, dev);
                tma_load_4d<true>(da + H_A_BYTES / 2, &tma_a, bar, m0 + 64, k0, piece, dev);
              } else {
                tma_load_4d<true>(da, &tma_a, bar, k0, m0, piece, dev);
              }
              uint8_t* db = b_hi(s) + piece * S::B_BYTES;
              if (args.b_k_major) {
                tma_load_4d<true>(db, &tma_b, bar, k0, nb0, piece, dev);
              } else {
#pragma unroll
                for (int c = 0; c < S::BNH / 64; ++c)
                  tma_load_4d<true>(db + c * 8192, &tma_b, bar, nb0 + 64 * c, k0, piece, dev);
              }
            }
          }
          __syncwarp();
        }
      }
    } else if (warp == 1 && crank == 0) {
      // ---------------- MMA issuer (leader CTA) ----------------
      // kind::f16 idesc: D f32 (bit 4), A/B fp16 (0), K- or MN-major per operand
      const uint32_t idesc = (1u << 4) | ((uint32_t)(args.a_mn_major ? 1 : 0) << 15) |
                             ((uint32_t)(args.b_k_major ? 0 : 1) << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)((HB * H_CG) >> 4) << 24);
      // SWIZZLE_128B descriptors: K-major rows of 128 B, 8-row groups 1 KB apart,
      // one k-step (16 fp16) = 32 B along the row; MN-major: 64-element MN
      // chunks (one TMA box, 8 KB) apart by LBO, 8-k groups by SBO, one k-step =
      // 16 rows of 128 B.
      const uint32_t a_lbo = args.a_mn_major ? 8192u : 16u;
      const uint32_t a_step = args.a_mn_major ? 2048u : 32u;
      const uint32_t b_lbo = args.b_k_major ? 16u : 8192u;
      const uint32_t b_step = args.b_k_major ? 32u : 2048u;
      const uint64_t da0 = smem_desc(smem_u32(a_hi(0)), a_lbo, 1024u, 2u);
      const uint64_t db0 = smem_desc(smem_u32(b_hi(0)), b_lbo, 1024u, 2u);
      const uint64_t dak = a_step >> 4, dbk = b_step >> 4;
      const uint64_t alo = H_A_BYTES >> 4, blo = S::B_BYTES >> 4;
      int rs = 0;
      uint32_t rph = 0;
      int cg = 0;
      for (int j = 0;; ++j) {
        const int u = get_unit(j, false);
        if (u >= args.units) break;
        int t, sp, c0, ncu;
        unit_of(u, t, sp, c0, ncu);
        const int kbe = min(nk, 2 * (c0 + ncu));
        for (int kb = 2 * c0; kb < kbe; ++kb) {
          const int kin = kb & 1;
          const int buf = cg & 1;
          const bool chunk_last = kin == 1 || kb == kbe - 1;
          if (kin == 0) mbar_wait<true>(&tempty[buf], ((cg >> 1) & 1) ^ 1);
          mbar_wait<true>(&raw_full[rs], rph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = da0 + (uint64_t)(rs * (S::STAGE >> 4));
          const uint64_t db = db0 + (uint64_t)(rs * (S::STAGE >> 4));
          const uint32_t dacc = tmem_d + (uint32_t)(buf * BN);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < HBK / 16; ++kk) {
              const uint64_t ah = da + kk * dak, bh = db + kk * dbk;
              mma_f16_ss<1>(dacc, ah, bh + blo, idesc, (kin | kk) ? 1u : 0u);   // hi.lo
              mma_f16_ss<2>(dacc, ah, bh, idesc, 1u);                           // hi.hi
              mma_f16_ss<0>(dacc, ah + alo, bh, idesc, 1u);                     // lo.hi
            }
            mma_commit<2>(&raw_empty[rs]);
            if (chunk_last) mma_commit<2>(&tfull[buf]);
          }
          __syncwarp();
          if (++rs == RS) { rs = 0; rph ^= 1u; }
          if (chunk_last) ++cg;
        }
      }
    }
  } else {
    // ---------------- drain: scaled fp32 promotion of every k chunk, C stores ----------------
    if (BN > 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    const int q = warp & 3;
    const int dg = (warp - 4) >> 2;            // column group: columns [128 dg, 128 dg + 128)
    int cg = 0;
    uint32_t fold_ph = 0;
    for (int j = 0;; ++j) {
      const int u = get_unit(j, false);
      if (u >= args.units) break;
      int t, sp, c0, ncu, m0, n0, dev;
      unit_of(u, t, sp, c0, ncu);
      tile_of(t, m0, n0, dev);
      m0 += (int)crank * HB;
      const int mblk = m0 / HB, nblk = (n0 + dg * 128) / HB;
      const float* sa = reinterpret_cast<const float*>(args.sa + (uint64_t)((int64_t)dev * args.sa_dev)) + mblk * args.sa_m;
      const float* sb = reinterpret_cast<const float*>(args.sb + (uint64_t)((int64_t)dev * args.sb_dev)) + nblk * args.sb_n;
      const bool live = mblk < args.rb_a && n0 + dg * 128 < args.N;
      float acc[128];
#pragma unroll
      for (int j = 0; j < 128; ++j) acc[j] = 0.f;
      for (int ci = 0; ci < ncu; ++ci, ++cg) {
        const int buf = cg & 1;
        const int c = c0 + ci;
        const float f = live ? __fmul_rn(sa[c * args.sa_k], sb[c * args.sb_k]) : 0.f;
        mbar_wait(&tfull[buf], (cg >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t v[32];
          tmem_ld32(tmem_d + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN + dg * 128 + cc * 32), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[cc * 32 + j] = __fmaf_rn(__uint_as_float(v[j]), f, acc[cc * 32 + j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          uint32_t r;
          asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(&tempty[buf])));
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
        }
      }
      const int row0 = m0 + q * 32;
      const int col0 = n0 + dg * 128;
      if (row0 >= args.M || col0 >= args.N) continue;
      uint8_t* stg = smem + S::STG_OFF + (warp - 4) * S::STG_WARP;
      constexpr int NSTG = S::STG_WARP / 4096;
      // one 32 x 128 slice (this warp's rows, its column group) through TMA
      // stores: 32 x 32 sub-slices via a 128B-swizzled staging tile
      auto store_slice = [&](const CUtensorMap* map, int row) {
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          if (col0 + cc * 32 >= args.N) break;
          uint8_t* tt = stg + (cc % NSTG) * 4096;
          if (cc >= NSTG) {
            if (lane == 0) {
              if (NSTG == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(tt + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_float4(acc[cc * 32 + 4 * j], acc[cc * 32 + 4 * j + 1], acc[cc * 32 + 4 * j + 2],
                            acc[cc * 32 + 4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                    reinterpret_cast<uint64_t>(map)),
                "r"(col0 + cc * 32), "r"(row), "r"(dev), "r"(smem_u32(tt))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      };
      if (BN == 128 && args.splits > 1) {
        // partial slice -> workspace; the last of the S units of this slice folds
        store_slice(&tma_w, sp * args.M + row0);
        uint32_t* flag = reinterpret_cast<uint32_t*>(args.flag_base + (uint64_t)((int64_t)dev * args.flag_dev)) +
                         (((int64_t)(t % (args.tiles_m * args.tiles_n)) * H_CG + crank) * S::NDG + dg) * 4 + q;
        uint32_t old = 0;
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(flag) : "memory");
        }
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old != (uint32_t)(args.splits - 1)) continue;
        if (args.fold_tma) {
          // last: the other S-1 partial slices come in by TMA (4 KB 32 x 32
          // boxes into the operand stages, idle now: a split GEMM gives every
          // pair one unit) and fold with this unit's own partial, in split order
          uint8_t* fbuf = smem + (warp - 4) * (12 * 4096);
          uint64_t* fb = &fold_bar[warp - 4];
          if (lane == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            mbar_expect_tx(fb, (uint32_t)((args.splits - 1) * 4 * 4096));
            int slot = 0;
            for (int s2 = 0; s2 < args.splits; ++s2) {
              if (s2 == sp) continue;
              for (int cc = 0; cc < 4; ++cc, ++slot)
                tma_load_3d(fbuf + slot * 4096, &tma_w, fb, col0 + cc * 32, s2 * args.M + row0, dev);
            }
          }
          __syncwarp();
          mbar_wait(fb, fold_ph);
          fold_ph ^= 1u;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 v;
              for (int s2 = 0; s2 < args.splits; ++s2) {
                float4 x;
                if (s2 == sp) {
                  x = make_float4(acc[cc * 32 + 4 * j], acc[cc * 32 + 4 * j + 1], acc[cc * 32 + 4 * j + 2],
                                  acc[cc * 32 + 4 * j + 3]);
                } else {
                  const int slot = (s2 < sp ? s2 : s2 - 1) * 4 + cc;
                  x = *reinterpret_cast<const float4*>(fbuf + slot * 4096 + lane * 128 + ((j ^ (lane & 7)) << 4));
                }
                if (s2 == 0) {
                  v = x;
                } else {
                  v.x = __fadd_rn(v.x, x.x); v.y = __fadd_rn(v.y, x.y);
                  v.z = __fadd_rn(v.z, x.z); v.w = __fadd_rn(v.w, x.w);
                }
              }
              acc[cc * 32 + 4 * j] = v.x; acc[cc * 32 + 4 * j + 1] = v.y;
              acc[cc * 32 + 4 * j + 2] = v.z; acc[cc * 32 + 4 * j + 3] = v.w;
            }
          store_slice(&tma_c, row0);
          if (lane == 0) *flag = 0u;          // consumed: ready for the next launch
          continue;
        }

        // last: fold the S partials in split order (own one re-read from L2)
        // straight from global to C: lane = column, every load and store one
        // 128-byte line (row-per-lane reads were L2-request bound)
        const float* ws = reinterpret_cast<const float*>(args.ws_base + (uint64_t)((int64_t)dev * args.ws_dev));
        float* cb = reinterpret_cast<float*>(args.c_base + (uint64_t)((int64_t)dev * args.dev_stride));
        const int64_t sst = (int64_t)args.M * args.N;
        // acc (already stored as this unit's partial) is reused as x[row][col
        // group]: every split's 128 lines per warp are in flight at once
        const int nrow = min(32, args.M - row0);
        const float* p0 = ws + (int64_t)row0 * args.N + col0 + lane;
#pragma unroll
        for (int r = 0; r < 32; ++r)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) acc[r * 4 + cc] = r < nrow ? __ldcg(p0 + (int64_t)r * args.N + cc * 32) : 0.f;
#pragma unroll 1
        for (int s2 = 1; s2 < args.splits; ++s2) {
          const float* ps = p0 + s2 * sst;
#pragma unroll
          for (int r = 0; r < 32; ++r)
#pragma unroll
            for (int cc = 0; cc < 4; ++cc)
              if (r < nrow) acc[r * 4 + cc] = __fadd_rn(acc[r * 4 + cc], __ldcg(ps + (int64_t)r * args.N + cc * 32));
        }
#pragma unroll
        for (int r = 0; r < 32; ++r)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            if (r < nrow) cb[(int64_t)(row0 + r) * args.ldc + col0 + cc * 32 + lane] = acc[r * 4 + cc];
        if (lane == 0) *flag = 0u;            // consumed: ready for the next launch
        continue;

      }
      if (args.tma_store) {
        store_slice(&tma_c, row0);
      } else {
        const int row = row0 + lane;
        if (row < args.M) {
          float* crow = reinterpret_cast<float*>(args.c_base + (uint64_t)((int64_t)dev * args.dev_stride)) +
                        (int64_t)row * args.ldc;
#pragma unroll
          for (int j = 0; j < 128; ++j)
            if (col0 + j < args.N) crow[col0 + j] = acc[j];
        }
      }
    }
    if (args.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "n"(S::TMEM_COLS));
  }
}

// 4-D fp16 pieces map {cols, rows, piece, device}, box {64, box_rows, 1, 1}, 128B swizzle.
int make_map_h16(CUtensorMap* map, uint64_t addr, uint64_t cols, uint64_t rows, uint64_t ndev, uint64_t pitch,
                 uint64_t dev_bytes, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return spx_set_error("cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {cols, rows, 2, ndev};
  cuuint64_t strides[3] = {pitch * 2, rows * pitch * 2, dev_bytes};
  cuuint32_t box[4] = {64, box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, reinterpret_cast<void*>(addr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return spx_set_error("cuTensorMapEncodeTiled (fp16 pieces) failed (%d)", (int)r);
  return 0;
}

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

void launch_split_args(const SplitArgs& a, int ndev, cudaStream_t s) {
  spx_launch(split_h16_kernel, dim3(H3_CL * ((a.cols + HB - 1) / HB), (a.rows + HB - 1) / HB, ndev), dim3(256), 0, s, a);
}

// Geometry of one operand's pieces: in the record's own workspace (offsets
// from its start, per-device strides of their own) or, shared, in the arena.
struct Operand {
  uint64_t src;
  int64_t ld;
  int rows, cols, rb, cb;
  int64_t pitch;                       // halves
  int64_t piece_off, scl_off;          // workspace offsets (bytes) or arena addresses (shared)
  int64_t piece_dev, scl_dev;          // bytes between devices
};

void operand_geom(Operand& o, uint64_t src, int64_t ld, int rows, int cols, int ndev, int64_t& ws) {
  o.src = src;
  o.ld = ld;
  o.rows = rows;
  o.cols = cols;
  o.rb = (rows + HB - 1) / HB;
  o.cb = (cols + HB - 1) / HB;
  o.pitch = align_up(cols, 8);
  o.piece_dev = align_up(2 * (int64_t)rows * o.pitch * 2, 1024);
  o.scl_dev = align_up((int64_t)o.rb * o.cb * 4, 256);
  o.piece_off = ws;
  ws += o.piece_dev * ndev;
  o.scl_off = ws;
  ws += o.scl_dev * ndev;
  ws = align_up(ws, 1024);
}

void split_args(SplitArgs& s, const Operand& o, int64_t src_dev, uint64_t ws) {
  s.src = o.src;
  s.src_dev = src_dev;
  s.ld = o.ld;
  s.rows = o.rows;
  s.cols = o.cols;
  s.dst = ws + (uint64_t)o.piece_off;
  s.dst_dev = o.piece_dev;
  s.pitch = o.pitch;
  s.scl = ws + (uint64_t)o.scl_off;
  s.scl_dev = o.scl_dev;
  s.cb = o.cb;
}

}  // namespace

struct SpxGemmH3 {
  spx_gemm_params p;
  uint32_t* sched = nullptr;            // dynamic-scheduling counters (H3Args::sched)
  Operand A, B;
  int64_t ws_bytes = 0;
  uint64_t ws = 0;
  CUtensorMap ma, mb, mc, mw;
  H3Args args;
  SplitArgs sa, sb;
  dim3 grid;
  int bn = 128;         // output columns per CTA pair (H3Cfg)
  int splits = 1;       // split-K units per tile
  int64_t part_off = 0; // split-K partials in the workspace (after the flag words at 0)
};

// Split-K flag words live at the start of every stream workspace (a fixed
// region, so no other GEMM's partials ever overwrite them): uint32
// [tiles][2][BN/128][4] per device, tiles <= SM pairs when split.
constexpr int64_t H3_FLAG_DEV = 8192;

bool spx_gemm_h3_supported(const spx_gemm_params& p) {
  return spx_gemm_tc_supported(p) && p.splits <= 1 && p.epi == SPX_EPI_NONE;
}

// BN and split count for one GEMM.  BN = 256 (the largest MMA, least
// shared-memory traffic per FLOP) unless its coarser tiles leave more of the
// last wave idle -- compared in waves of CTA pairs, a BN = 256 tile costing
// ~0.95 of two BN = 128 tiles.  Split-K when the tiles fill at most half the
// pairs: S units per tile, each >= 2 k chunks (256 of K).
static void h3_shape(const spx_gemm_params& p, int& bn, int& splits) {
  const int sms = spx_num_sms() - (p.reserve_sms > 0 ? p.reserve_sms : 0);
  const int pairs = sms / H_CG > 0 ? sms / H_CG : 1;
  const int64_t tm = (p.M + HB * H_CG - 1) / (HB * H_CG);
  const int64_t t128 = tm * ((p.N + 127) / 128) * p.ndev, t256 = tm * ((p.N + 255) / 256) * p.ndev;
  const double w128 = (double)((t128 + pairs - 1) / pairs), w256 = (double)((t256 + pairs - 1) / pairs);
  // a BN = 256 tile costs ~0.85 of two BN = 128 tiles on this power-capped board:
  // the 256-wide MMA reads 52 instead of 73 B/cycle of operands from shared
  // memory and half the B traffic from L2, and the energy saved raises the
  // clock (C3 N=1 +2.7%, profiles/r02_c3_n1_variants.txt)
  static double c256 = -1;
  if (c256 < 0) {
    const char* e = getenv("SPX_H3_BN256_COST");
    c256 = e ? atof(e) : 0.85;
  }
  bn = (p.N > 128 && w256 * 2 * c256 < w128) ? 256 : 128;
  if (const char* e = getenv("SPX_H3_BN")) bn = atoi(e) == 256 ? 256 : 128;
  const int64_t tiles = bn == 256 ? t256 : t128;
  const int nch = (int)(((p.K + HBK - 1) / HBK + 1) / 2);
  // off by default.  Measured (profiles/r01_gemm_h3_splitk.txt): long-K GEMMs
  // gain (512x1024x4096: 44 -> 36 us) but short ones lose (512x1024x1024:
  // 19 -> 27 us: partial stores + counter + fold ~8 us), and whole C2 steps at
  // N=2/4 get 2-6% slower even with forward-only splits; SPX_H3_SPLITK=n (or
  // h3_splitk = n > 1) enables up to n splits
  int maxs = p.h3_splitk > 1 ? p.h3_splitk : 1;
  if (const char* e = getenv("SPX_H3_SPLITK"))
    if (p.h3_splitk != 1) maxs = atoi(e);
  splits = 1;
  const uint64_t cb = p.base + (uint64_t)(p.c_off * 4);
  const bool tma_ok = (cb & 15) == 0 && (p.ldc & 3) == 0 && (p.dev_stride & 15) == 0 && p.ldc == p.N;
  if (maxs > 1 && bn == 128 && tma_ok && p.M % 32 == 0 && p.N % 128 == 0 && tiles * 2 <= pairs &&
      tiles * H_CG * 2 * 4 * 4 <= H3_FLAG_DEV) {
    int sk = (int)(pairs / tiles);
    sk = sk < nch / 2 ? sk : nch / 2;
    sk = sk < maxs ? sk : maxs;
    splits = sk > 1 ? sk : 1;
  }
}

int spx_gemm_h3_prepare(const spx_gemm_params& p, SpxGemmH3** out) {
  if (!spx_gemm_h3_supported(p)) return spx_set_error("gemm %dx%dx%d: block-scaled fp16 path unsupported", p.M, p.N, p.K);
  SpxGemmH3* g = new SpxGemmH3();
  g->p = p;
  const uint64_t a = p.base + (uint64_t)(p.a_off * 4), b = p.base + (uint64_t)(p.b_off * 4);
  h3_shape(p, g->bn, g->splits);
  int64_t ws = 0;
  if (g->splits > 1) {
    ws = H3_FLAG_DEV * p.ndev;
    g->part_off = ws;
    ws += align_up((int64_t)g->splits * p.M * p.N * 4, 1024) * p.ndev;
  }
  if (p.a_mn_major) operand_geom(g->A, a, p.lda, p.K, p.M, p.ndev, ws);
  else operand_geom(g->A, a, p.lda, p.M, p.K, p.ndev, ws);
  if (p.b_k_major) operand_geom(g->B, b, p.ldb, p.N, p.K, p.ndev, ws);
  else operand_geom(g->B, b, p.ldb, p.K, p.N, p.ndev, ws);
  if (p.h3_shared) {
    // pieces and scales live in the arena, written by SPX_K_SPLIT records
    auto shared = [&](Operand& o, int64_t off, int64_t scl) {
      o.piece_off = (int64_t)(p.base + (uint64_t)(off * 4));
      o.scl_off = (int64_t)(p.base + (uint64_t)(scl * 4));
      o.piece_dev = o.scl_dev = p.dev_stride;
    };
    shared(g->A, p.h3_a_off, p.h3_a_scl);
    shared(g->B, p.h3_b_off, p.h3_b_scl);
    ws = g->splits > 1 ? g->part_off + align_up((int64_t)g->splits * p.M * p.N * 4, 1024) * p.ndev : 0;
  }
  g->ws_bytes = ws;
  *out = g;
  return 0;
}

int64_t spx_gemm_h3_ws_bytes(const SpxGemmH3* g) { return g->ws_bytes; }

int spx_gemm_h3_bind(SpxGemmH3* g, uint64_t ws) {
  const spx_gemm_params& p = g->p;
  if (!ws && g->ws_bytes) return spx_set_error("gemm h3: workspace not bound");
  const uint64_t wsb = ws;            // the stream workspace (split-K flags + partials)
  if (p.h3_shared) ws = 0;            // operand addresses are absolute
  g->ws = wsb ? wsb : 1;
  const Operand &A = g->A, &B = g->B;
  if (make_map_h16(&g->ma, ws + A.piece_off, A.cols, A.rows, p.ndev, A.pitch, A.piece_dev, p.a_mn_major ? 64 : HB))
    return -1;
  if (make_map_h16(&g->mb, ws + B.piece_off, B.cols, B.rows, p.ndev, B.pitch, B.piece_dev,
                   p.b_k_major ? g->bn / H_CG : 64))
    return -1;
  split_args(g->sa, A, p.dev_stride, ws);
  split_args(g->sb, B, p.dev_stride, ws);
  H3Args& a_ = g->args;
  a_.M = p.M; a_.N = p.N; a_.K = p.K;
  a_.a_mn_major = p.a_mn_major;
  a_.b_k_major = p.b_k_major;
  a_.tiles_m = (p.M + HB * H_CG - 1) / (HB * H_CG);
  a_.tiles_n = (p.N + g->bn - 1) / g->bn;
  a_.tiles = a_.tiles_m * a_.tiles_n * p.ndev;
  {
    // concurrent tiles ~ pairs: a group_m x (pairs / group_m) rectangle, A panels
    // 256 rows, B panels BN columns (same K): footprint minimal at
    // group_m = sqrt(pairs * BN / 256).  SPX_H3_GROUP_M=n forces n (0: M fastest)
    int sms = spx_num_sms() - (p.reserve_sms > 0 ? p.reserve_sms : 0);
    const double pairs = sms / H_CG > 0 ? sms / H_CG : 1;
    int gm = (int)(sqrt(pairs * g->bn / 256.0) + 0.5);
    if (const char* e = getenv("SPX_H3_GROUP_M")) gm = atoi(e);
    if (gm <= 0 || gm > a_.tiles_m) gm = a_.tiles_m;
    a_.group_m = gm;
  }
  a_.c_base = p.base + (uint64_t)(p.c_off * 4);
  a_.dev_stride = p.dev_stride;
  a_.ldc = p.ldc;
  a_.sa = ws + (uint64_t)A.scl_off;
  a_.sb = ws + (uint64_t)B.scl_off;
  a_.sa_dev = A.scl_dev;
  a_.sb_dev = B.scl_dev;
  // A stored [M][K]: scales [m-block][k-block]; stored [K][M]: [k-block][m-block]
  a_.sa_m = p.a_mn_major ? 1 : A.cb;
  a_.sa_k = p.a_mn_major ? A.cb : 1;
  a_.sb_n = p.b_k_major ? B.cb : 1;
  a_.sb_k = p.b_k_major ? 1 : B.cb;
  a_.rb_a = (p.M + HB - 1) / HB;
  a_.tma_store = 0;
  const char* e = getenv("SPX_GEMM_TMA_STORE");
  if (!(e && e[0] == '0') && (a_.c_base & 15) == 0 && (p.ldc & 3) == 0 && (p.dev_stride & 15) == 0) {
    if (make_map(&g->mc, a_.c_base, p.N, p.M, p.ndev, p.ldc * 4, p.dev_stride, 32, false)) return -1;
    a_.tma_store = 1;
  } else {
    memset(&g->mc, 0, sizeof(g->mc));
  }
  a_.splits = g->splits;
  a_.units = a_.tiles * g->splits;
  {
    static int dyn = -1;
    if (dyn < 0) {
      const char* e = getenv("SPX_H3_DYNAMIC");
      dyn = e ? atoi(e) != 0 : 1;
    }
    a_.dyn = dyn;
    if (dyn && !g->sched) {
      SPX_CUDA(cudaMalloc(&g->sched, 8));
      SPX_CUDA(cudaMemset(g->sched, 0, 8));
    }
    a_.sched = reinterpret_cast<uint64_t>(g->sched);
    static int ft = -1;
    if (ft < 0) {
      const char* e = getenv("SPX_H3_FOLD_TMA");
      ft = e ? atoi(e) != 0 : 1;
    }
    // the TMA fold stages the other S-1 partial slices (4 boxes of 4 KB each)
    // in the drain warp's 48 KB share of the operand stages: S <= 4; more
    // splits (long-K weight gradients) fold straight from global memory
    a_.fold_tma = ft && (g->splits - 1) * 4 * 4096 <= 12 * 4096;
  }
  memset(&g->mw, 0, sizeof(g->mw));
  a_.flag_base = wsb;
  a_.flag_dev = H3_FLAG_DEV;
  a_.ws_base = wsb + (uint64_t)g->part_off;
  a_.ws_dev = align_up((int64_t)g->splits * p.M * p.N * 4, 1024);
  if (g->splits > 1) {
    if (!a_.tma_store) return spx_set_error("gemm h3 %dx%dx%d: split-K needs TMA stores", p.M, p.N, p.K);
    if (make_map(&g->mw, a_.ws_base, p.N, (uint64_t)p.M * g->splits, p.ndev, (uint64_t)p.N * 4, a_.ws_dev, 32, false))
      return -1;
    SPX_CUDA(cudaMemset(reinterpret_cast<void*>(wsb), 0, (size_t)(H3_FLAG_DEV * p.ndev)));
  }
  int sms = spx_num_sms() - (p.reserve_sms > 0 ? p.reserve_sms : 0);
  sms -= sms % H_CG;
  if (sms < H_CG) sms = H_CG;
  const int want = a_.units * H_CG;
  g->grid = dim3((unsigned)(want < sms ? want : sms));
  return 0;
}

template <int BN>
static cudaError_t launch_h3(const SpxGemmH3* g, cudaStream_t s) {
  using S = H3Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_h3_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g->grid;
  cfg.blockDim = dim3(S::THREADS);
  cfg.dynamicSmemBytes = S::TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = H_CG;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  if (spx_pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, gemm_h3_kernel<BN>, g->ma, g->mb, g->mc, g->mw, g->args);
}

int spx_gemm_h3_launch(const SpxGemmH3* g, cudaStream_t s, int* nlaunch) {
  const spx_gemm_params& p = g->p;
  if (!g->ws) return spx_set_error("gemm h3: workspace not bound");
  if (!p.h3_shared) {
    launch_split_args(g->sa, p.ndev, s);
    SPX_CHECK_LAUNCH();
    launch_split_args(g->sb, p.ndev, s);
    SPX_CHECK_LAUNCH();
    if (nlaunch) *nlaunch += 2;
  }
  if (g->bn == 256) SPX_CUDA(launch_h3<256>(g, s));
  else SPX_CUDA(launch_h3<128>(g, s));

  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

static int split_args(const spx_split_params& p, SplitArgs& a) {
  if (p.rows <= 0 || p.cols <= 0 || (p.pitch & 7) || p.pitch < p.cols)
    return spx_set_error("split: bad geometry %dx%d pitch %lld", p.rows, p.cols, (long long)p.pitch);
  a.src = p.base + (uint64_t)(p.src_off * 4);
  a.src_dev = p.dev_stride;
  a.ld = p.ld;
  a.rows = p.rows;
  a.cols = p.cols;
  a.dst = p.base + (uint64_t)(p.dst_off * 4);
  a.dst_dev = p.dev_stride;
  a.pitch = p.pitch;
  a.scl = p.base + (uint64_t)(p.scl_off * 4);
  a.scl_dev = p.dev_stride;
  a.cb = (p.cols + HB - 1) / HB;
  return 0;
}

int spx_launch_split(const spx_split_params& p, cudaStream_t s, int* nlaunch) {
  SplitArgs a;
  if (split_args(p, a)) return -1;
  launch_split_args(a, p.ndev, s);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

int spx_split_batch_max(void) { return SPLIT_MAX_JOBS; }

int spx_launch_split_batch(const spx_split_params* const* p, int n, cudaStream_t s, int* nlaunch) {
  if (n < 1 || n > SPLIT_MAX_JOBS) return spx_set_error("split batch: %d jobs (1..%d)", n, SPLIT_MAX_JOBS);
  SplitBatch b;
  memset(&b, 0, sizeof(b));
  b.n = n;
  int64_t total = 0;
  for (int j = 0; j < n; ++j) {
    if (p[j]->ndev != p[0]->ndev) return spx_set_error("split batch: device counts differ");
    if (split_args(*p[j], b.job[j])) return -1;
    b.start[j] = (int)total;
    total += (int64_t)b.job[j].cb * ((p[j]->rows + HB - 1) / HB);
  }
  b.start[n] = (int)total;
  if (total * H3_CL > INT32_MAX) return spx_set_error("split batch: grid too large");
  spx_launch(split_h16_batch_kernel, dim3((unsigned)(total * H3_CL), p[0]->ndev, 1), dim3(256), 0, s, b);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

int spx_h3_range_split(uint32_t* out, int reset) {
  SPX_CUDA(cudaMemcpyFromSymbol(out, g_h3_range_split, sizeof(uint32_t)));
  if (reset && *out) {
    const uint32_t z = 0;
    SPX_CUDA(cudaMemcpyToSymbol(g_h3_range_split, &z, sizeof(z)));
  }
  return 0;
}

void spx_gemm_h3_free(SpxGemmH3* g) {
  if (g->sched) cudaFree(g->sched);
  delete g;
}
