// tcgen05 / TMEM / TMA GEMM for the reference's fp32 `matmul`
// (interp.py:43-44: numpy `@` on float32 arrays -> sgemm).
//
// fp32 parity (<= 1e-5 max-normalised error) on tensor cores uses
// the 3xTF32 split: x = hi + lo, hi = x truncated to the tf32 grid, lo = x - hi
// (exact in fp32), and  A.B ~= hi(A).hi(B) + hi(A).lo(B) + lo(A).hi(B).
// Measured on B200 (tools/tf32_conversion.py): kind::tf32 ignores the low 13
// mantissa bits of an fp32 operand, i.e. it truncates -- so the raw TMA tile
// already IS hi(x) and the split only writes lo(x).
//
// Tensor-core accumulation is not IEEE round-to-nearest: measured error grows
// linearly with K (3e-5 at K=4096).  Each CTA therefore accumulates `promote`
// k-blocks per TMEM chunk and folds finished chunks into fp32 registers
// (__fadd_rn) while the tensor core fills the other chunk buffer; hi.hi and the
// two correction terms go to separate accumulators (independent MMA chains --
// one accumulator serialised the MMAs).  Error 7e-7..8e-7 at any K.
//
// Persistent kernel, one CTA per SM, 128 x 128 output tiles.  (A CTA-pair
// variant with tcgen05.mma.cta_group::2 M=256 was measured slower on these
// shapes -- the cross-CTA split/drain handshakes sat on the critical path --
// and was dropped.)  Warp roles (10 warps):
//   warp 0      TMA producer into a RSTAGES-deep raw ring (k-slab of 32 fp32)
//   warp 1      TMEM alloc; MMA issuer: per k-step of 8
//               hi.lo (A collector fill), hi.hi (collector reuse), lo.hi
//   warps 2..5  split: lo = x - trunc_tf32(x) into a LSTAGES-deep lo ring
//   warps 6..9  drain: TMEM -> registers fp32 promotion, epilogue stores
// Transposed operands (a `transpose` feeding the matmul) are loaded MN-major
// (SWIZZLE_128B_BASE32B, the only MN-major layout tf32 accepts), so the
// transpose never materialises (interp.py:51-52 folded into the descriptor).
// The third dimension of the TMA tensor maps walks co-located mesh devices.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <cstring>
#include "common.cuh"
#include "tc_util.cuh"

namespace {

constexpr int BM = 128;             // rows per CTA
constexpr int BN = 128;             // output columns per CTA (= per pair)
constexpr int BK = 32;              // fp32 elements per 128-byte swizzle row
constexpr int NTHREADS = 320;
constexpr int NTHREADS_T = 512;   // TMEM-A kernel: 4 warpgroups

struct TcArgs {
  int M, N, K, a_mn_major, b_k_major, promote;   // promote: k-blocks per TMEM chunk
  int tiles_m, tiles_n, tiles;                   // persistent tile space (x ndev)
  int splits, units;                             // split-K: units = tiles x splits
  uint64_t c_base;     // device 0 address of C
  int64_t dev_stride;  // bytes
  int64_t ldc;
  // fused epilogue (spx_gemm_params.epi*): offsets in elements from base
  uint64_t base;
  int tma_store;       // plain C stores through the tensor map (else row stores)
  int sk_inkernel;     // split-K partials reduced in the kernel (spx_gemm_params.sk_mode)
  uint64_t ws_base, flag_base;
  int epi;
  int64_t in_off[2], in_ld[2], out_off[2], out_ld[2];
  float imm[2];
};

// One accumulator value through the fused epilogue (spindle_b200.h,
// spx_epilogue) -- the same IEEE operations, in the same order, as the
// elementwise kernel it replaces (ew.cu / interp.cuh).
template <int EPI>
SPX_DEV void epi_apply(float c, float x0, float x1, float k0, float k1, float& y0, float& y1) {
  if (EPI == SPX_EPI_ADD) {
    y0 = f_add(x0, c);
  } else if (EPI == SPX_EPI_SQUARE) {
    y0 = c;
    y1 = f_mul(c, c);
  } else if (EPI == SPX_EPI_MULSCALE) {
    y0 = f_mul(c, f_mul(x0, k0));
  } else if (EPI == SPX_EPI_MOMENTUM) {
    y0 = f_add(f_mul(x0, k0), c);
    y1 = f_add(x1, -f_mul(y0, k1));
  }
}

// Epilogue of one drain warp: its 32 accumulator rows (lane = row, acc[] =
// the BN columns) go through a padded 32 x 33 shared-memory tile per 32-column
// chunk, so that afterwards lane = column and every global load/store of the
// warp is one 128-byte row segment (row-per-lane stores hit 32 lines each).
template <int EPI>
SPX_DEV void epi_store_tile(const TcArgs& a, int dev, int sp, int row0, int n0, const float* acc, float* stg,
                            int lane) {
  constexpr int NIN = EPI == SPX_EPI_ADD || EPI == SPX_EPI_MULSCALE ? 1 : EPI == SPX_EPI_MOMENTUM ? 2 : 0;
  constexpr int NOUT = EPI == SPX_EPI_SQUARE || EPI == SPX_EPI_MOMENTUM ? 2 : 1;
  constexpr int EG = NIN >= 2 ? 8 : 16;   // rows per group: loads of a group in flight together
  float* db = reinterpret_cast<float*>(a.base + (uint64_t)((int64_t)dev * a.dev_stride));
  const int rows = min(32, a.M - row0);
#pragma unroll
  for (int cc = 0; cc < BN / 32; ++cc) {
    const int col = n0 + cc * 32 + lane;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = acc[cc * 32 + j];
    __syncwarp();
    if (col >= a.N) continue;
#pragma unroll 1
    for (int r0 = 0; r0 < rows; r0 += EG) {
      float c[EG], x0[EG], x1[EG];
#pragma unroll
      for (int r = 0; r < EG; ++r) {
        const int64_t row = row0 + r0 + r;
        c[r] = stg[(r0 + r) * 33 + lane];
        if (r0 + r < rows) {
          if (NIN >= 1) x0[r] = db[a.in_off[0] + row * a.in_ld[0] + col];
          if (NIN >= 2) x1[r] = db[a.in_off[1] + row * a.in_ld[1] + col];
        }
      }
#pragma unroll
      for (int r = 0; r < EG; ++r) {
        if (r0 + r >= rows) break;
        const int64_t row = row0 + r0 + r;
        if (EPI == SPX_EPI_NONE) {
          reinterpret_cast<float*>(a.c_base + (uint64_t)((int64_t)dev * a.dev_stride))[((int64_t)sp * a.M + row) * a.ldc + col] = c[r];
          continue;
        }
        float y0, y1 = 0.f;
        epi_apply<EPI>(c[r], NIN >= 1 ? x0[r] : 0.f, NIN >= 2 ? x1[r] : 0.f, a.imm[0], a.imm[1], y0, y1);
        db[a.out_off[0] + row * a.out_ld[0] + col] = y0;
        if (NOUT == 2) db[a.out_off[1] + row * a.out_ld[1] + col] = y1;
      }
    }
  }
}

// Work unit u -> (tile t, split s) and its k-block range [kb0, kb0 + nku).
SPX_DEV void unit_range(const TcArgs& a, int nk, int u, int& t, int& s, int& kb0, int& nku) {
  t = u / a.splits;
  s = u - t * a.splits;
  kb0 = (int)(((long long)nk * s) / a.splits);
  nku = (int)(((long long)nk * (s + 1)) / a.splits) - kb0;
}

SPX_DEV void tile_coords(const TcArgs& a, int t, int& m0, int& n0, int& dev, int bm = BM) {
  const int per_dev = a.tiles_m * a.tiles_n;
  dev = t / per_dev;
  const int r = t - dev * per_dev;
  const int n_blk = r / a.tiles_m;            // M fastest: concurrent CTAs share B panels
  m0 = (r - n_blk * a.tiles_m) * bm;
  n0 = n_blk * BN;
}

// ---------------------------------------------------------------------------
// Variant with the A operand in TENSOR MEMORY (tcgen05.mma ... [a_tmem] ...).
// The split warps read each A row from the TMA'd smem tile (any layout, one
// lane per row = one TMEM lane), write hi(A) and lo(A) into TMEM with
// tcgen05.st, and only lo(B) goes back to smem: the tensor core then reads
// just B from shared memory (3 x 4 KB per k-step instead of 5 x 4 KB), the
// split writes half as many smem bytes.  Per 128x128x32 k-block the smem
// traffic falls from ~176 KB to ~128 KB (the kernel above is smem-bound).
// TMEM: [0,256) two chunk accumulators (one chain each), [256, 256+64*LS)
// the A hi/lo stages.
// ---------------------------------------------------------------------------
SPX_DEV void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

template <int CG>
SPX_DEV void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  if (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

template <int RS_, int LS_, int CG_ = 1>
struct CfgT {
  static constexpr int CG = CG_;                    // CTAs per tile (tcgen05 cta_group)
  static constexpr int BNH = BN / CG;               // B rows (output columns) this CTA holds
  static constexpr int A_BYTES = BM * BK * 4;       // 16 KB
  static constexpr int B_BYTES = BNH * BK * 4;      // 16 KB (8 KB per CTA of a pair)
  static constexpr int RAW = A_BYTES + B_BYTES;
  static constexpr int RSTAGES = RS_;
  static constexpr int LSTAGES = LS_;
  static constexpr int LO_OFF = RSTAGES * RAW;      // lo(B) ring
  static constexpr int BAR_OFF = LO_OFF + LSTAGES * B_BYTES;
  // epilogue staging per drain warp: two 32 x 32 fp32 tiles (128B-swizzled
  // TMA-store sources), or one 32 x 33 transpose tile for fused epilogues
  static constexpr int STG_OFF = (BAR_OFF + 256 + 1023) / 1024 * 1024;
  static constexpr int STG_WARP = 8192;
  static constexpr int TOTAL = STG_OFF + 4 * STG_WARP + 1024;
  static constexpr int TMEM_A = 2 * BN;             // first A column
};

template <int RS_, int LS_, int CG, int EPI>
__global__ void __launch_bounds__(NTHREADS_T, 1)
gemm_tc_tmema_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                     const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ CUtensorMap tma_w,
                     const __grid_constant__ TcArgs args) {
  using S = CfgT<RS_, LS_, CG>;
  constexpr int RS = S::RSTAGES, LS = S::LSTAGES;
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned base kept as __shared__ pointer arithmetic, so the split
  // warps' accesses compile to LDS/STS rather than generic loads
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* raw_empty = raw_full + RS;
  uint64_t* lo_full = raw_empty + RS;
  uint64_t* lo_empty = lo_full + LS;
  uint64_t* tfull = lo_empty + LS;
  uint64_t* tempty = tfull + 2;
  uint64_t* skbar = tempty + 2;          // [4] in-kernel split-K: partial tiles landed (per drain warp)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(skbar + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (args.K + BK - 1) / BK;
  // CG == 2: a cluster of two CTAs computes one 256 x 128 tile with
  // tcgen05.mma.cta_group::2 issued by rank 0.  Each CTA holds its own 128 A
  // rows (TMEM) and half of the B tile (64 output columns, smem), and drains
  // its own 128 x 128 accumulator.  Per SM this halves the tensor core's B
  // reads from shared memory and a quarter of the L2->SM traffic.
  uint32_t crank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int pair0 = blockIdx.x / CG, npairs = gridDim.x / CG;
  // arrive on rank 0's copy of a barrier (the MMA issuer's)
  auto arrive_leader = [&](uint64_t* bar) {
    if (CG == 1) {
      mbar_arrive(bar);
    } else {
      uint32_t r;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(bar)));
      // default semantics (as CUTLASS's ClusterBarrier::arrive): an explicit
      // .release.cluster costs ~1000 cycles of the issuing warp
      asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
    }
  };
  const int P = args.promote;

  auto a_raw = [&](int s) { return smem + s * S::RAW; };
  auto b_hi = [&](int s) { return smem + s * S::RAW + S::A_BYTES; };
  auto b_lo = [&](int s) { return smem + S::LO_OFF + s * S::B_BYTES; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], 1);
    }
    for (int s = 0; s < LS; ++s) {
      mbar_init(&lo_full[s], 4 * CG);             // one elected lane per split warp
      mbar_init(&lo_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4 * CG);              // one elected lane per drain warp
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&skbar[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 1) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 1) __syncthreads();
  else asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_d = *tmem_slot;
  SPX_PDL_ENTRY();   // barrier init, TMEM alloc, descriptor prefetch overlap the previous kernel

  // Warpgroup roles (setmaxnreg moves registers to the drain warpgroup, whose
  // fp32 promotion accumulators hold a 32 x 128 tile slice per warp):
  //   WG0  warp 0 TMA producer, warp 1 MMA issuer, warps 2-3 idle   (56 regs)
  //   WG1, WG2  split, alternating k-blocks (g & 1)                 (104 regs)
  //   WG3  drain + epilogue                                         (240 regs)
  // One split warpgroup per k-block left the tensor core waiting on the
  // split ~1/3 of the time; two alternating groups give each 2 k-blocks of
  // MMA time per k-block of split work.
  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (warp == 0) {
    // ---------------- TMA producer ----------------
    int g = 0;
    for (int u = pair0; u < args.units; u += npairs) {
      int t, sp, kb0, nku, m0, n0, dev;
      unit_range(args, nk, u, t, sp, kb0, nku);
      tile_coords(args, t, m0, n0, dev, BM * CG);
      m0 += (int)crank * BM;
      const int nb0 = n0 + (int)crank * S::BNH;
      for (int kb = 0; kb < nku; ++kb, ++g) {
        const int s = g % RS;
        mbar_wait(&raw_empty[s], ((g / RS) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&raw_full[s], (uint32_t)S::RAW);
          const int k0 = (kb0 + kb) * BK;
          if (args.a_mn_major) {
#pragma unroll
            for (int c = 0; c < BM / 32; ++c)
              tma_load_3d(a_raw(s) + c * 4096, &tma_a, &raw_full[s], m0 + 32 * c, k0, dev);
          } else {
            tma_load_3d(a_raw(s), &tma_a, &raw_full[s], k0, m0, dev);
          }
          if (args.b_k_major) {
            tma_load_3d(b_hi(s), &tma_b, &raw_full[s], k0, nb0, dev);
          } else {
#pragma unroll
            for (int c = 0; c < S::BNH / 32; ++c)
              tma_load_3d(b_hi(s) + c * 4096, &tma_b, &raw_full[s], nb0 + 32 * c, k0, dev);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 && crank == 0) {
    // ---------------- MMA issuer ----------------
    // One warp issues for the whole CTA, so its per-k-block instruction count
    // bounds the tensor core: everything except the waits is precomputed or
    // advanced incrementally (stage/phase counters, descriptors as base +
    // offset -- the address field is the low 14 bits of the descriptor, and
    // every smem address here is < 256 KB, so adding never carries out).
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) |
                           ((uint32_t)(args.b_k_major ? 0 : 1) << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)((BM * CG) >> 4) << 24);
    const uint32_t b_lbo = args.b_k_major ? 16u : 4096u, b_step = args.b_k_major ? 32u : 1024u;
    const uint32_t b_sbo = args.b_k_major ? 1024u : 512u;
    const uint32_t b_lay = args.b_k_major ? 2u : 1u;
    const uint64_t dbh0 = smem_desc(smem_u32(b_hi(0)), b_lbo, b_sbo, b_lay);
    const uint64_t dbl0 = smem_desc(smem_u32(b_lo(0)), b_lbo, b_sbo, b_lay);
    const uint64_t dkk = b_step >> 4;
    int rs = 0, ls = 0, cg = 0;
    uint32_t lph = 0;
    for (int u = pair0; u < args.units; u += npairs) {
      int t, sp, kb0, nku;
      unit_range(args, nk, u, t, sp, kb0, nku);
      int kin = 0;                                  // k-block index inside the chunk
      for (int kb = 0; kb < nku; ++kb) {
        const int buf = cg & 1;
        const bool chunk_last = kin == P - 1 || kb == nku - 1;
        if (kin == 0) {
          mbar_wait<CG == 2>(&tempty[buf], ((cg >> 1) & 1) ^ 1);
        }
        mbar_wait<CG == 2>(&lo_full[ls], lph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t dbh = dbh0 + (uint64_t)(rs * (S::RAW >> 4));
        const uint64_t dbl = dbl0 + (uint64_t)(ls * (S::B_BYTES >> 4));
        const uint32_t dacc = tmem_d + (uint32_t)(buf * BN);
        const uint32_t ahi = tmem_d + (uint32_t)(S::TMEM_A + ls * 64), alo = ahi + 32;
        const uint32_t init = kin == 0 ? 0u : 1u;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            mma_tf32_ts<CG>(dacc, ahi + kk * 8, dbl + kk * dkk, idesc, kk == 0 ? init : 1u);   // hi.lo
            mma_tf32_ts<CG>(dacc, alo + kk * 8, dbh + kk * dkk, idesc, 1u);                    // lo.hi
            mma_tf32_ts<CG>(dacc, ahi + kk * 8, dbh + kk * dkk, idesc, 1u);                    // hi.hi
          }
          mma_commit<CG>(&raw_empty[rs]);                 // CG == 2: both CTAs' barriers
          mma_commit<CG>(&lo_empty[ls]);
          if (chunk_last) mma_commit<CG>(&tfull[buf]);
        }
        __syncwarp();
        if (++rs == RS) rs = 0;
        if (++ls == LS) { ls = 0; lph ^= 1u; }
        if (chunk_last) { kin = 0; ++cg; } else { ++kin; }
      }
    }
  }
  } else if (warp < 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 112;");
    // ---------------- split: A rows -> TMEM (hi, lo); lo(B) -> smem ----------------
    const int q = warp & 3;                       // TMEM lane quadrant = A rows 32q..32q+31
    const int row = q * 32 + lane;
    const int grp = (warp - 4) >> 2;              // k-blocks g with (g & 1) == grp
    const int t0 = (threadIdx.x - 128) & 127;     // 0..127 for the B part
    int g = 0;
    for (int u = pair0; u < args.units; u += npairs) {
      int t, sp, kb0, nku;
      unit_range(args, nk, u, t, sp, kb0, nku);
      for (int kb = 0; kb < nku; ++kb, ++g) {
        if ((g & 1) != grp) continue;
        const int rs = g % RS, ls = g % LS;
        mbar_wait(&raw_full[rs], (g / RS) & 1);
        mbar_wait(&lo_empty[ls], ((g / LS) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // A row `row`: 32 consecutive k values
        uint32_t hi[32], lo[32];
        const float* abase = reinterpret_cast<const float*>(a_raw(rs));
        if (args.a_mn_major) {
          // [mchunk][k][32 m], 32B-granule swizzle: granule g' = g ^ (k & 3)
          const int mc = row >> 5, mm = row & 31;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int gran = (mm >> 3) ^ (k & 3);
            const float x = abase[mc * 1024 + k * 32 + gran * 8 + (mm & 7)];
            hi[k] = __float_as_uint(x);
          }
        } else {
          // [m][32 k], 16B-chunk swizzle: chunk c' = c ^ (m & 7)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = *reinterpret_cast<const float4*>(abase + row * 32 + ((c ^ (row & 7)) << 2));
            hi[4 * c] = __float_as_uint(x.x); hi[4 * c + 1] = __float_as_uint(x.y);
            hi[4 * c + 2] = __float_as_uint(x.z); hi[4 * c + 3] = __float_as_uint(x.w);
          }
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float x = __uint_as_float(hi[k]);
          lo[k] = __float_as_uint(x - __uint_as_float(hi[k] & 0xFFFFE000u));
        }
        const uint32_t ta = tmem_d + ((uint32_t)(q * 32) << 16) + (uint32_t)(S::TMEM_A + ls * 64);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        // lo(B) into smem (same swizzled layout as the raw tile)
        const float4* src = reinterpret_cast<const float4*>(b_hi(rs));
        float4* dst = reinterpret_cast<float4*>(b_lo(ls));
#pragma unroll 4
        for (int i = t0; i < S::B_BYTES / 16; i += 128) {
          const float4 x = src[i];
          dst[i] = make_float4(x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u),
                               x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u),
                               x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u),
                               x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive_leader(&lo_full[ls]);
      }
    }
  } else {
    // ---------------- drain + epilogue ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    const int q = warp & 3;
    int cg = 0;
    for (int u = pair0; u < args.units; u += npairs) {
      int t, sp, kb0, nku, m0, n0, dev;
      unit_range(args, nk, u, t, sp, kb0, nku);
      tile_coords(args, t, m0, n0, dev, BM * CG);
      m0 += (int)crank * BM;
      const int nchunks = (nku + P - 1) / P;
      if (EPI == SPX_EPI_ADD || EPI == SPX_EPI_MULSCALE || EPI == SPX_EPI_MOMENTUM) {
        // pull the epilogue's input rows into L2 while the tile accumulates
        const int prow = m0 + q * 32 + lane;
        if (prow < args.M) {
          const char* db = reinterpret_cast<const char*>(args.base + (uint64_t)((int64_t)dev * args.dev_stride));
#pragma unroll
          for (int i = 0; i < (EPI == SPX_EPI_MOMENTUM ? 2 : 1); ++i) {
            const char* rp = db + 4 * (args.in_off[i] + (int64_t)prow * args.in_ld[i] + n0);
#pragma unroll
            for (int l = 0; l < BN * 4 / 128; ++l)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + 128 * l));
          }
        }
      }
      float acc[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) acc[j] = 0.f;
      for (int c = 0; c < nchunks; ++c, ++cg) {
        const int buf = cg & 1;
        mbar_wait(&tfull[buf], (cg >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc) {
          uint32_t v[32];
          tmem_ld32(tmem_d + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN + cc * 32), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[cc * 32 + j] = __fadd_rn(acc[cc * 32 + j], __uint_as_float(v[j]));
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive_leader(&tempty[buf]);
      }
      const int row = m0 + q * 32 + lane;
      if (EPI == SPX_EPI_SQUARE) {
        // no inputs: row per lane, 16 B stores of C and C * C
        if (row < args.M) {
          float* db = reinterpret_cast<float*>(args.base + (uint64_t)((int64_t)dev * args.dev_stride));
          float* o0 = db + args.out_off[0] + (int64_t)row * args.out_ld[0];
          float* o1 = db + args.out_off[1] + (int64_t)row * args.out_ld[1];
          const bool vec = ((args.out_off[0] | args.out_off[1] | args.out_ld[0] | args.out_ld[1] | n0) & 3) == 0;
#pragma unroll
          for (int cc = 0; cc < BN / 32; ++cc) {
            const int col0 = n0 + cc * 32;
            if (vec && col0 + 32 <= args.N) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float* ac = acc + cc * 32 + 4 * j;
                *reinterpret_cast<float4*>(o0 + col0 + 4 * j) = make_float4(ac[0], ac[1], ac[2], ac[3]);
                *reinterpret_cast<float4*>(o1 + col0 + 4 * j) =
                    make_float4(f_mul(ac[0], ac[0]), f_mul(ac[1], ac[1]), f_mul(ac[2], ac[2]), f_mul(ac[3], ac[3]));
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j < args.N) {
                  o0[col0 + j] = acc[cc * 32 + j];
                  o1[col0 + j] = f_mul(acc[cc * 32 + j], acc[cc * 32 + j]);
                }
            }
          }
        }
      } else if (EPI != SPX_EPI_NONE) {
        // fused epilogue: loads of its inputs want coalesced rows (transpose)
        float* stg = reinterpret_cast<float*>(smem + S::STG_OFF + q * S::STG_WARP);
        if (m0 + q * 32 < args.M) epi_store_tile<EPI>(args, dev, sp, m0 + q * 32, n0, acc, stg, lane);
      } else if (args.tma_store) {
        // plain store through TMA: each 32-row x 32-column slice goes to a
        // 128B-swizzled staging tile (conflict-free float4 writes, lane = row)
        // and leaves the SM as one bulk tensor store
        uint8_t* stg = smem + S::STG_OFF + q * S::STG_WARP;
        const bool rows_in = m0 + q * 32 < args.M;
        // in-kernel split-K: split s > 0 stores its partial slice into the
        // workspace and counts it into the slice's flag; split 0 waits for the
        // other splits, folds their partials in split order, then stores C
        const bool sk = args.sk_inkernel && args.splits > 1;
        uint32_t* flag = reinterpret_cast<uint32_t*>(args.flag_base + (uint64_t)((int64_t)dev * args.dev_stride)) +
                         ((int64_t)t * CG + crank) * 4 + q;
        const bool to_ws = sk && sp > 0;
        const CUtensorMap* map = to_ws ? &tma_w : &tma_c;
        const int rowc = to_ws ? (sp - 1) * args.M + m0 + q * 32 : (sk ? 0 : sp * args.M) + m0 + q * 32;
        if (sk && sp == 0 && rows_in) {
          if (lane == 0) {
            const uint32_t want = (uint32_t)(args.splits - 1);
            const long long t0 = clock64();
            uint32_t v;
            for (;;) {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
              if (v >= want) break;
              __nanosleep(64);
              if (clock64() - t0 > 20000000000LL) __trap();
            }
          }
          __syncwarp();
          // The CTA's only work unit is done (units <= CTA pairs), so its raw
          // TMA ring is idle: bring every partial slice of this warp's 32 rows
          // in with bulk tensor loads (128B-swizzled 32 x 32 boxes), then fold
          // them in split order from shared memory.
          uint8_t* ring = smem + q * (S::RSTAGES * S::RAW / 4);
          int nbox = 0;
          for (int cc = 0; cc < BN / 32; ++cc)
            if (n0 + cc * 32 < args.N) ++nbox;
          if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&skbar[q], (uint32_t)((args.splits - 1) * nbox * 4096));
            for (int s2 = 1; s2 < args.splits; ++s2)
              for (int cc = 0; cc < nbox; ++cc)
                tma_load_3d(ring + ((s2 - 1) * 4 + cc) * 4096, &tma_w, &skbar[q], n0 + cc * 32,
                            (s2 - 1) * args.M + m0 + q * 32, dev);
          }
          mbar_wait(&skbar[q], 0);
          for (int s2 = 1; s2 < args.splits; ++s2) {
#pragma unroll
            for (int cc = 0; cc < BN / 32; ++cc) {
              if (cc >= nbox) break;
              const uint8_t* box = ring + ((s2 - 1) * 4 + cc) * 4096 + lane * 128;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 w = *reinterpret_cast<const float4*>(box + ((j ^ (lane & 7)) << 4));
                acc[cc * 32 + 4 * j] = __fadd_rn(acc[cc * 32 + 4 * j], w.x);
                acc[cc * 32 + 4 * j + 1] = __fadd_rn(acc[cc * 32 + 4 * j + 1], w.y);
                acc[cc * 32 + 4 * j + 2] = __fadd_rn(acc[cc * 32 + 4 * j + 2], w.z);
                acc[cc * 32 + 4 * j + 3] = __fadd_rn(acc[cc * 32 + 4 * j + 3], w.w);
              }
            }
          }
          __syncwarp();
          if (lane == 0) *flag = 0u;      // consumed: ready for the next launch
        }
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc) {
          // every staged slice is stored and committed as one bulk group, so
          // wait_group.read 1 below really frees the buffer of slice cc - 2
          if (!rows_in || n0 + cc * 32 >= args.N) break;
          uint8_t* t = stg + (cc & 1) * 4096;
          if (cc >= 2) {
            // the store issued from this buffer two slices ago must have read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(t + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_float4(acc[cc * 32 + 4 * j], acc[cc * 32 + 4 * j + 1], acc[cc * 32 + 4 * j + 2],
                            acc[cc * 32 + 4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                    reinterpret_cast<uint64_t>(map)),
                "r"(n0 + cc * 32), "r"(rowc), "r"(dev), "r"(smem_u32(t))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (to_ws && rows_in) {
          // the partial must be in memory before the owner is told
          if (lane == 0) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
          }
          __syncwarp();
        }
        // staging is reused by the next tile: all of this tile's stores must have read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      } else if (row < args.M) {
        // plain store: row per lane, 16 B per access (fire-and-forget)
        float* crow = reinterpret_cast<float*>(args.c_base + (uint64_t)((int64_t)dev * args.dev_stride)) +
                      ((int64_t)sp * args.M + row) * args.ldc;
#pragma unroll
        for (int cc = 0; cc < BN / 32; ++cc) {
          const int col0 = n0 + cc * 32;
          if (col0 + 32 <= args.N && (args.ldc & 3) == 0) {
            float4* dst = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[j] = make_float4(acc[cc * 32 + 4 * j], acc[cc * 32 + 4 * j + 1], acc[cc * 32 + 4 * j + 2],
                                   acc[cc * 32 + 4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < args.N) crow[col0 + j] = acc[cc * 32 + j];
          }
        }
      }
    }
  }
  if (warp >= 12 && args.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // CG == 2: neither CTA leaves while its peer may still arrive on its barriers
  // or the pair's MMAs may still read its shared memory / TMEM
  if (CG == 1) __syncthreads();
  else asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_d));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_d));
  }
}

}  // namespace

struct SpxGemmTC {
  CUtensorMap ma, mb, mc, mw;
  TcArgs args;
  dim3 grid;
  int cg;              // CTAs per tile (1, or 2 = cluster pair with cta_group::2 MMAs)
  spx_gemm_params p;
};

bool spx_gemm_tc_supported(const spx_gemm_params& p) {
  // TMA: 16B-aligned base and row pitch; tile sizes make tiny shapes a waste.
  const uint64_t da = p.base + (uint64_t)(p.a_off * 4), db = p.base + (uint64_t)(p.b_off * 4);
  if ((da & 15) || (db & 15) || (p.lda & 3) || (p.ldb & 3) || (p.dev_stride & 15)) return false;
  if (p.M < 64 || p.N < 32 || p.K < 32) return false;
  return true;
}

int spx_gemm_tc_prepare(const spx_gemm_params& p, SpxGemmTC** out) {
  SpxGemmTC* g = new SpxGemmTC();
  g->p = p;
  { const char* e = getenv("SPX_GEMM_CG"); g->cg = e ? atoi(e) : 2; }
  if (g->cg != 1) g->cg = 2;
  const uint64_t a = p.base + (uint64_t)(p.a_off * 4), b = p.base + (uint64_t)(p.b_off * 4);
  int rc;
  if (p.a_mn_major) rc = make_map(&g->ma, a, p.M, p.K, p.ndev, p.lda * 4, p.dev_stride, 32, true);
  else rc = make_map(&g->ma, a, p.K, p.M, p.ndev, p.lda * 4, p.dev_stride, BM, false);
  if (rc) { delete g; return rc; }
  if (p.b_k_major) rc = make_map(&g->mb, b, p.K, p.N, p.ndev, p.ldb * 4, p.dev_stride, BN / g->cg, false);
  else rc = make_map(&g->mb, b, p.N, p.K, p.ndev, p.ldb * 4, p.dev_stride, 32, true);
  if (rc) { delete g; return rc; }
  TcArgs& a_ = g->args;
  a_.M = p.M; a_.N = p.N; a_.K = p.K;
  a_.a_mn_major = p.a_mn_major; a_.b_k_major = p.b_k_major;
  { const char* e = getenv("SPX_GEMM_PROMOTE"); a_.promote = p.promote > 0 ? p.promote : (e ? atoi(e) : 4); }
  a_.tiles_m = (p.M + BM * g->cg - 1) / (BM * g->cg);
  a_.tiles_n = (p.N + BN - 1) / BN;
  a_.tiles = a_.tiles_m * a_.tiles_n * p.ndev;
  a_.splits = p.splits > 1 ? p.splits : 1;
  a_.units = a_.tiles * a_.splits;
  a_.c_base = p.base + (uint64_t)(p.c_off * 4);
  a_.dev_stride = p.dev_stride;
  a_.ldc = p.ldc;
  a_.base = p.base;
  a_.epi = p.epi;
  // TMA stores of C: 16B-aligned base and pitch; with split-K the partial
  // slabs are stacked rows, so a 32-row box must not straddle two of them
  a_.tma_store = 0;
  {
    const char* e = getenv("SPX_GEMM_TMA_STORE");
    const bool want = !(e && e[0] == '0');
    const bool ok = (a_.c_base & 15) == 0 && (p.ldc & 3) == 0 && (p.dev_stride & 15) == 0 &&
                    (a_.splits == 1 || p.M % 32 == 0);
    if (want && ok && p.epi == SPX_EPI_NONE) {
      const uint64_t rows = (uint64_t)p.M * (p.sk_mode == 1 ? 1 : a_.splits);
      if (make_map(&g->mc, a_.c_base, p.N, rows, p.ndev, p.ldc * 4, p.dev_stride, 32, false)) {
        delete g;
        return -1;
      }
      a_.tma_store = 1;
    }
  }
  if (!a_.tma_store) memset(&g->mc, 0, sizeof(g->mc));
  memset(&g->mw, 0, sizeof(g->mw));
  a_.sk_inkernel = 0;
  if (p.sk_mode == 1 && a_.splits > 1) {
    const int pairs = (spx_num_sms() - (p.reserve_sms > 0 ? p.reserve_sms : 0)) / g->cg;
    if (!a_.tma_store || p.N != p.ldc || p.M % 32 || a_.units > pairs) {
      delete g;
      return spx_set_error("gemm %dx%dx%d: in-kernel split-K needs TMA stores, ldc == N, M %% 32 == 0 and "
                           "units <= SM pairs (%d > %d)", p.M, p.N, p.K, a_.units, pairs);
    }
    a_.sk_inkernel = 1;
    a_.ws_base = p.base + (uint64_t)(p.ws_off * 4);
    a_.flag_base = p.base + (uint64_t)(p.flag_off * 4);
    if (make_map(&g->mw, a_.ws_base, p.N, (uint64_t)p.M * (a_.splits - 1), p.ndev, (uint64_t)p.N * 4,
                 p.dev_stride, 32, false)) {
      delete g;
      return -1;
    }
  }
  for (int i = 0; i < 2; ++i) {
    a_.in_off[i] = p.epi_in_off[i];
    a_.in_ld[i] = p.epi_in_ld[i];
    a_.out_off[i] = p.epi_out_off[i];
    a_.out_ld[i] = p.epi_out_ld[i];
    a_.imm[i] = p.epi_imm[i];
  }
  if (p.epi != SPX_EPI_NONE && p.splits > 1) {
    delete g;
    return spx_set_error("gemm: fused epilogue with split-K");
  }
  int sms = spx_num_sms() - (p.reserve_sms > 0 ? p.reserve_sms : 0);
  sms -= sms % g->cg;
  if (sms < g->cg) sms = g->cg;
  const int want = a_.units * g->cg;
  g->grid = dim3((unsigned)(want < sms ? want : sms));
  *out = g;
  return 0;
}

template <int RS_, int LS_, int CG, int EPI>
static int launch_tmema_e(const SpxGemmTC* g, cudaStream_t s) {
  static bool attr = false;
  auto kern = gemm_tc_tmema_kernel<RS_, LS_, CG, EPI>;
  if (!attr) {
    SPX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgT<RS_, LS_, CG>::TOTAL));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g->grid;
  cfg.blockDim = dim3(NTHREADS_T);
  cfg.dynamicSmemBytes = CfgT<RS_, LS_, CG>::TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (CG > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = CG;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (spx_pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  SPX_CUDA(cudaLaunchKernelEx(&cfg, kern, g->ma, g->mb, g->mc, g->mw, g->args));
  return 0;
}

// one kernel instantiation per epilogue (a single kernel holding every
// epilogue variant was measured slower: its code crowded the other roles)
template <int RS_, int LS_, int CG>
static int launch_tmema(const SpxGemmTC* g, cudaStream_t s) {
  switch (g->args.epi) {
    case SPX_EPI_ADD: return launch_tmema_e<RS_, LS_, CG, SPX_EPI_ADD>(g, s);
    case SPX_EPI_SQUARE: return launch_tmema_e<RS_, LS_, CG, SPX_EPI_SQUARE>(g, s);
    case SPX_EPI_MULSCALE: return launch_tmema_e<RS_, LS_, CG, SPX_EPI_MULSCALE>(g, s);
    case SPX_EPI_MOMENTUM: return launch_tmema_e<RS_, LS_, CG, SPX_EPI_MOMENTUM>(g, s);
    default: return launch_tmema_e<RS_, LS_, CG, SPX_EPI_NONE>(g, s);
  }
}

int spx_gemm_tc_launch(const SpxGemmTC* g, cudaStream_t s, int* nlaunch) {
  static int pipe = -1;
  if (pipe < 0) {
    const char* e = getenv("SPX_GEMM_PIPE");
    pipe = e ? atoi(e) : 0;
  }
  int rc;
  if (g->cg == 2) {
    switch (pipe) {
      case 53: rc = launch_tmema<5, 3, 2>(g, s); break;
      default: rc = launch_tmema<6, 4, 2>(g, s);
    }
  } else {
    switch (pipe) {
      default: rc = launch_tmema<4, 4, 1>(g, s);
    }
  }
  if (rc) return rc;
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

void spx_gemm_tc_free(SpxGemmTC* g) { delete g; }
