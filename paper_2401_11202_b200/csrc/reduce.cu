// Reduction over any subset of dims (interp.py:53-55: np.sum / np.max with
// axis=dims), with the reduced operand given as a fused elementwise program,
// so e.g. the loss `reduce(mul(d, d), [0, 1])` reads `d` once.
//
// The host permutes the operand so kept dims come first and reduced dims
// last (x.dims = kept ++ reduced), then collapses each group.  Element (o, r)
// is output o, reduction index r.  Two-pass and deterministic: pass 1 folds a
// fixed chunk of r per (chunk, o) into scratch, pass 2 folds the chunks in
// order.  Thread mappings keep loads coalesced and 16B wide:
//   ROW  (reduced dim innermost)  a warp per output, lanes walk r (float4)
//   COL  (kept dim innermost)     a lane per 4 consecutive outputs (float4),
//                                 8 row groups walk r, smem combine
//   GEN  any other rank/stride pattern, scalar
#include <cfloat>
#include "interp.cuh"

namespace {

SPX_DEV float ident(int monoid) { return monoid == 0 ? 0.f : -INFINITY; }
SPX_DEV float fold(int monoid, float a, float b) { return monoid == 0 ? f_add(a, b) : f_max(a, b); }

SPX_DEV float* out_ptr(const spx_reduce_params& p, int d, int nchunks, int c, int64_t o) {
  return nchunks == 1 ? dev_ptr(p.x.base, p.x.dev_stride, d, p.out_off) + o
                      : dev_ptr(p.x.base, p.x.dev_stride, d, p.scratch_off) + (int64_t)c * p.n_out + o;
}

// 2-D loads: value of view j at (o, r..r+W-1) [ROW] or (o..o+W-1, r) [COL].
template <int W, bool ROW>
SPX_DEV void load2d(const spx_reduce_params& p, const float* fb, int64_t o, int64_t r, RegFile<W>& f) {
  const spx_ew_params& x = p.x;
  const int ro = p.n_kept == 1 ? 0 : -1;     // dim index of o (if any)
  const int rr = p.n_kept;                   // dim index of r
#pragma unroll
  for (int j = 0; j < SPX_MAX_IN; ++j) {
    if (j >= x.n_in) break;
    const int64_t so = ro >= 0 ? x.in[j].stride[0] : 0;
    const int64_t sr = x.in[j].stride[rr];
    const int64_t off = x.in[j].off + o * so + r * sr;
    const int64_t sfast = ROW ? sr : so;
    if (W == 4 && sfast == 1) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(fb + off));
      f.r[j].v[0] = v.x; f.r[j].v[1 % W] = v.y; f.r[j].v[2 % W] = v.z; f.r[j].v[3 % W] = v.w;
    } else if (sfast == 0 || W == 1) {
      const float v = __ldg(fb + off);
#pragma unroll
      for (int k = 0; k < W; ++k) f.r[j].v[k] = v;
    } else {
#pragma unroll
      for (int k = 0; k < W; ++k) f.r[j].v[k] = __ldg(fb + off + k * sfast);
    }
  }
}

// WPO warps per output: 1 (8 outputs per block) or 8 (few outputs, e.g. the
// loss: the whole block walks one output's chunk, partials combined in smem
// in warp order)
template <int W, int WPO>
__global__ void __launch_bounds__(256) reduce_row(const __grid_constant__ spx_reduce_params p, int64_t chunk,
                                                  int nchunks) {
  SPX_PDL_ENTRY();
  __shared__ float part[8];
  const int d = blockIdx.z;
  const float* fb = dev_ptr(p.x.base, p.x.dev_stride, d, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t o = (int64_t)blockIdx.x * (8 / WPO) + warp / WPO;
  const int sub = warp % WPO;
  const int c = blockIdx.y;
  if (o >= p.n_out) return;
  const int64_t r0 = c * chunk, r1 = min(p.n_red_elems, r0 + chunk);
  float acc = ident(p.monoid);
  for (int64_t r = r0 + (int64_t)(sub * 32 + lane) * W; r < r1; r += 32 * W * WPO) {
    RegFile<W> f;
    load2d<W, true>(p, fb, o, r, f);
    run_program<W>(p.x.prog, p.x.imm, p.x.n_prog, f);
    const Vec<W> y = f.get(p.x.out_reg[0]);
#pragma unroll
    for (int k = 0; k < W; ++k) acc = fold(p.monoid, acc, y.v[k]);
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) acc = fold(p.monoid, acc, __shfl_xor_sync(0xffffffffu, acc, m));
  if (WPO == 1) {
    if (lane == 0) *out_ptr(p, d, nchunks, c, o) = acc;
    return;
  }
  if (lane == 0) part[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = part[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) v = fold(p.monoid, v, part[w]);
    *out_ptr(p, d, nchunks, c, o) = v;
  }
}

template <int W>
__global__ void __launch_bounds__(256) reduce_col(const __grid_constant__ spx_reduce_params p, int64_t chunk,
                                                  int nchunks) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.z;
  const float* fb = dev_ptr(p.x.base, p.x.dev_stride, d, 0);
  const int64_t o = ((int64_t)blockIdx.x * 32 + threadIdx.x) * W;
  const int c = blockIdx.y;
  const int64_t r0 = c * chunk, r1 = min(p.n_red_elems, r0 + chunk);
  Vec<W> acc;
#pragma unroll
  for (int k = 0; k < W; ++k) acc.v[k] = ident(p.monoid);
  if (o < p.n_out) {
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      RegFile<W> f;
      load2d<W, false>(p, fb, o, r, f);
      run_program<W>(p.x.prog, p.x.imm, p.x.n_prog, f);
      const Vec<W> y = f.get(p.x.out_reg[0]);
#pragma unroll
      for (int k = 0; k < W; ++k) acc.v[k] = fold(p.monoid, acc.v[k], y.v[k]);
    }
  }
  __shared__ float sm[8][32 * W + 1];
#pragma unroll
  for (int k = 0; k < W; ++k) sm[threadIdx.y][threadIdx.x * W + k] = acc.v[k];
  __syncthreads();
  if (threadIdx.y == 0 && o < p.n_out) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      float v = sm[0][threadIdx.x * W + k];
#pragma unroll
      for (int y = 1; y < 8; ++y) v = fold(p.monoid, v, sm[y][threadIdx.x * W + k]);
      if (o + k < p.n_out) *out_ptr(p, d, nchunks, c, o + k) = v;
    }
  }
}

// Generic: any rank; one warp per output, lanes walk r.
__global__ void __launch_bounds__(256) reduce_gen(const __grid_constant__ spx_reduce_params p, int64_t chunk,
                                                  int nchunks) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.z;
  const float* fb = dev_ptr(p.x.base, p.x.dev_stride, d, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t o = (int64_t)blockIdx.x * 8 + warp;
  const int c = blockIdx.y;
  if (o >= p.n_out) return;
  const spx_ew_params& x = p.x;
  const int64_t r0 = c * chunk, r1 = min(p.n_red_elems, r0 + chunk);
  float acc = ident(p.monoid);
  for (int64_t r = r0 + lane; r < r1; r += 32) {
    int64_t off[SPX_MAX_IN];
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j) off[j] = x.in[j].off;
    int64_t oo = o, rr = r;
#pragma unroll
    for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
      if (k >= x.rank) continue;
      int64_t idx;
      if (k >= p.n_kept) {
        if (k == p.n_kept) { idx = rr; } else { idx = rr % x.dims[k]; rr /= x.dims[k]; }
      } else {
        if (k == 0) { idx = oo; } else { idx = oo % x.dims[k]; oo /= x.dims[k]; }
      }
#pragma unroll
      for (int j = 0; j < SPX_MAX_IN; ++j) off[j] += idx * x.in[j].stride[k];
    }
    RegFile<1> f;
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j) {
      if (j >= x.n_in) break;
      f.r[j].v[0] = __ldg(fb + off[j]);
    }
    run_program<1>(x.prog, x.imm, x.n_prog, f);
    acc = fold(p.monoid, acc, f.get(x.out_reg[0]).v[0]);
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) acc = fold(p.monoid, acc, __shfl_xor_sync(0xffffffffu, acc, m));
  if (lane == 0) *out_ptr(p, d, nchunks, c, o) = acc;
}

// OUT mapping (mode 3): many outputs, few reduced elements (pooling windows,
// gradients of broadcasts): a thread owns 4 consecutive outputs along the
// contiguous innermost kept dim and walks the whole reduced range.
__global__ void __launch_bounds__(256) reduce_out(const __grid_constant__ spx_reduce_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const float* fb = dev_ptr(p.x.base, p.x.dev_stride, d, 0);
  float* out = dev_ptr(p.x.base, p.x.dev_stride, d, p.out_off);
  const spx_ew_params& x = p.x;
  const int nk = p.n_kept;
  for (int64_t o4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o4 * 4 < p.n_out;
       o4 += (int64_t)gridDim.x * blockDim.x) {
    int64_t base[SPX_MAX_IN];
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j) base[j] = x.in[j].off;
    int64_t rem = o4 * 4;
#pragma unroll
    for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
      if (k >= nk) continue;
      const int64_t ik = k == 0 ? rem : rem % x.dims[k];
      rem = k == 0 ? 0 : rem / x.dims[k];
#pragma unroll
      for (int j = 0; j < SPX_MAX_IN; ++j) base[j] += ik * x.in[j].stride[k];
    }
    Vec<4> acc;
#pragma unroll
    for (int q = 0; q < 4; ++q) acc.v[q] = ident(p.monoid);
    for (int64_t r = 0; r < p.n_red_elems; ++r) {
      RegFile<4> f;
      int64_t rr = r;
      int64_t roff[SPX_MAX_IN];
#pragma unroll
      for (int j = 0; j < SPX_MAX_IN; ++j) roff[j] = base[j];
#pragma unroll
      for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
        if (k < nk || k >= x.rank) continue;
        const int64_t ik = k == nk ? rr : rr % x.dims[k];
        rr = k == nk ? 0 : rr / x.dims[k];
#pragma unroll
        for (int j = 0; j < SPX_MAX_IN; ++j) roff[j] += ik * x.in[j].stride[k];
      }
#pragma unroll
      for (int j = 0; j < SPX_MAX_IN; ++j) {
        if (j >= x.n_in) break;
        if (x.in[j].stride[nk - 1] == 1) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(fb + roff[j]));
          f.r[j].v[0] = t.x; f.r[j].v[1] = t.y; f.r[j].v[2] = t.z; f.r[j].v[3] = t.w;
        } else {
          const float t = __ldg(fb + roff[j]);
          f.r[j].v[0] = t; f.r[j].v[1] = t; f.r[j].v[2] = t; f.r[j].v[3] = t;
        }
      }
      run_program<4>(x.prog, x.imm, x.n_prog, f);
      const Vec<4> y = f.get(x.out_reg[0]);
#pragma unroll
      for (int q = 0; q < 4; ++q) acc.v[q] = fold(p.monoid, acc.v[q], y.v[q]);
    }
    *reinterpret_cast<float4*>(out + o4 * 4) = make_float4(acc.v[0], acc.v[1], acc.v[2], acc.v[3]);
  }
}

// few outputs, many chunks: a block per output, strided fold + fixed smem tree
__global__ void __launch_bounds__(256) reduce_final_block(const __grid_constant__ spx_reduce_params p, int nchunks) {
  SPX_PDL_ENTRY();
  __shared__ float red[256];
  const int d = blockIdx.y;
  const int64_t o = blockIdx.x;
  const float* part = dev_ptr(p.x.base, p.x.dev_stride, d, p.scratch_off);
  float v = ident(p.monoid);
  for (int c = threadIdx.x; c < nchunks; c += 256) v = fold(p.monoid, v, part[(int64_t)c * p.n_out + o]);
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fold(p.monoid, red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) dev_ptr(p.x.base, p.x.dev_stride, d, p.out_off)[o] = red[0];
}

// OUT mapping for a plain view (one input, no elementwise program, <= 64
// reduced elements: the pooling windows of the U-Net analog): the reduced
// offsets do not depend on the output, so they are computed once per block
// into shared memory, and every thread issues all loads of a window before
// folding them (in r order, as reduce_out).  The generic kernel recomputed
// them with 64-bit divisions per element and loaded one element at a time.
constexpr int OUTV_MAX_RED = 64;
__global__ void __launch_bounds__(256) reduce_out_view(const __grid_constant__ spx_reduce_params p) {
  __shared__ int64_t sred[OUTV_MAX_RED];
  const spx_ew_params& x = p.x;
  const int nk = p.n_kept;
  const int nred = (int)p.n_red_elems;
  for (int r = threadIdx.x; r < nred; r += blockDim.x) {
    int64_t rr = r, off = 0;
#pragma unroll
    for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
      if (k < nk || k >= x.rank) continue;
      const int64_t ik = k == nk ? rr : rr % x.dims[k];
      rr = k == nk ? 0 : rr / x.dims[k];
      off += ik * x.in[0].stride[k];
    }
    sred[r] = off;
  }
  __syncthreads();
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const float* fb = dev_ptr(x.base, x.dev_stride, d, 0);
  float* out = dev_ptr(x.base, x.dev_stride, d, p.out_off);
  const bool v4 = x.in[0].stride[nk - 1] == 1;
  for (int64_t o4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o4 * 4 < p.n_out;
       o4 += (int64_t)gridDim.x * blockDim.x) {
    int64_t base = x.in[0].off;
    int64_t rem = o4 * 4;
#pragma unroll
    for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
      if (k >= nk) continue;
      const int64_t ik = k == 0 ? rem : rem % x.dims[k];
      rem = k == 0 ? 0 : rem / x.dims[k];
      base += ik * x.in[0].stride[k];
    }
    const float* src = fb + base;
    float4 acc = make_float4(ident(p.monoid), ident(p.monoid), ident(p.monoid), ident(p.monoid));
    for (int r0 = 0; r0 < nred; r0 += 8) {
      float4 t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (r0 + u < nred) {
          if (v4) {
            t[u] = __ldg(reinterpret_cast<const float4*>(src + sred[r0 + u]));
          } else {
            const float v = __ldg(src + sred[r0 + u]);
            t[u] = make_float4(v, v, v, v);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (r0 + u < nred) {
          acc.x = fold(p.monoid, acc.x, t[u].x);
          acc.y = fold(p.monoid, acc.y, t[u].y);
          acc.z = fold(p.monoid, acc.z, t[u].z);
          acc.w = fold(p.monoid, acc.w, t[u].w);
        }
      }
    }
    *reinterpret_cast<float4*>(out + o4 * 4) = acc;
  }
}

__global__ void reduce_final(const __grid_constant__ spx_reduce_params p, int nchunks) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const float* part = dev_ptr(p.x.base, p.x.dev_stride, d, p.scratch_off);
  float* out = dev_ptr(p.x.base, p.x.dev_stride, d, p.out_off);
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < p.n_out;
       o += (int64_t)gridDim.x * blockDim.x) {
    float v = part[o];
    for (int c = 1; c < nchunks; ++c) v = fold(p.monoid, v, part[(int64_t)c * p.n_out + o]);
    out[o] = v;
  }
}

}  // namespace

// p.mode: 0 ROW (2-D), 1 COL (2-D), 2 GEN; p.x.vec: float4 along the fast dim.
int spx_launch_reduce(const spx_reduce_params& p, cudaStream_t s, int* nlaunch) {
  if (p.n_out <= 0 || p.x.ndev <= 0) return 0;
  const int mode = p.mode;
  if (mode == 3) {
    int64_t b = (p.n_out / 4 + 255) / 256;
    const int64_t cap = (int64_t)spx_num_sms() * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    const bool view = p.x.n_in == 1 && p.x.n_prog == 0 && p.x.out_reg[0] == 0 && p.n_red_elems <= OUTV_MAX_RED;
    if (view) spx_launch(reduce_out_view, dim3((unsigned)b, (unsigned)p.x.ndev), 256, 0, s, p);
    else spx_launch(reduce_out, dim3((unsigned)b, (unsigned)p.x.ndev), 256, 0, s, p);
    SPX_CHECK_LAUNCH();
    if (nlaunch) ++*nlaunch;
    return 0;
  }
  const int W = p.x.vec ? 4 : 1;
  const bool few = mode == 0 && p.n_out < 64;        // ROW with a handful of outputs
  int64_t per_block_out = mode == 1 ? 32 * W : (few ? 1 : 8);
  const int64_t out_blocks = (p.n_out + per_block_out - 1) / per_block_out;
  const int64_t target = (int64_t)spx_num_sms() * 4;
  int64_t nchunks = (target + out_blocks * p.x.ndev - 1) / (out_blocks * p.x.ndev);
  const int64_t min_chunk = mode == 1 ? 64 : 2048;
  const int64_t max_chunks = (p.n_red_elems + min_chunk - 1) / min_chunk;
  if (nchunks > max_chunks) nchunks = max_chunks;
  if (nchunks < 1) nchunks = 1;
  if (nchunks > 1 && p.scratch_off < 0) nchunks = 1;
  if (nchunks > 4096) nchunks = 4096;
  int64_t chunk = (p.n_red_elems + nchunks - 1) / nchunks;
  if (mode == 0) chunk = (chunk + 127) / 128 * 128;      // keep float4 lanes aligned
  nchunks = (p.n_red_elems + chunk - 1) / chunk;
  if (nchunks < 1) nchunks = 1;
  dim3 grid((unsigned)out_blocks, (unsigned)nchunks, (unsigned)p.x.ndev);
  if (mode == 0) {
    if (few) {
      if (W == 4) spx_launch(reduce_row<4, 8>, grid, 256, 0, s, p, chunk, (int)nchunks);
      else spx_launch(reduce_row<1, 8>, grid, 256, 0, s, p, chunk, (int)nchunks);
    } else {
      if (W == 4) spx_launch(reduce_row<4, 1>, grid, 256, 0, s, p, chunk, (int)nchunks);
      else spx_launch(reduce_row<1, 1>, grid, 256, 0, s, p, chunk, (int)nchunks);
    }
  } else if (mode == 1) {
    if (W == 4) spx_launch(reduce_col<4>, grid, dim3(32, 8), 0, s, p, chunk, (int)nchunks);
    else spx_launch(reduce_col<1>, grid, dim3(32, 8), 0, s, p, chunk, (int)nchunks);
  } else {
    spx_launch(reduce_gen, grid, 256, 0, s, p, chunk, (int)nchunks);
  }
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  if (nchunks > 1 && p.n_out < 64 && nchunks >= 64) {
    spx_launch(reduce_final_block, dim3((unsigned)p.n_out, (unsigned)p.x.ndev), 256, 0, s, p, (int)nchunks);
    SPX_CHECK_LAUNCH();
    if (nlaunch) ++*nlaunch;
  } else if (nchunks > 1) {
    int64_t b = (p.n_out + 255) / 256;
    if (b > 1024) b = 1024;
    spx_launch(reduce_final, dim3((unsigned)b, (unsigned)p.x.ndev), 256, 0, s, p, (int)nchunks);
    SPX_CHECK_LAUNCH();
    if (nlaunch) ++*nlaunch;
  }
  return 0;
}
