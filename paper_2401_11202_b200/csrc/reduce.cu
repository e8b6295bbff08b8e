// Reduction over any subset of dims (interp.py:53-55: np.sum / np.max with
// axis=dims), with the reduced operand given as a fused elementwise
// expression, so e.g. the loss `reduce(mul(d, d), [0, 1])` reads `d` once.
//
// The host permutes the operand so the kept dims come first and the reduced
// dims last (x.dims = kept ++ reduced); element (o, r) of the permuted operand
// is output o, reduction index r.  Two-pass and deterministic: pass 1 folds
// fixed chunks of r per (chunk, o) into scratch, pass 2 folds the chunks in
// order.  Two thread mappings keep global loads coalesced:
//   COL  the operand's innermost dim is kept -> lanes walk consecutive o
//   ROW  the innermost dim is reduced        -> lanes walk consecutive r
#include <cfloat>
#include "common.cuh"

namespace {

SPX_DEV float ident(int monoid) { return monoid == 0 ? 0.f : -INFINITY; }
SPX_DEV float fold(int monoid, float a, float b) { return monoid == 0 ? f_add(a, b) : f_max(a, b); }

// Evaluate the reduced expression at permuted multi-index (o, r).
SPX_DEV float eval_at(const spx_reduce_params& p, const float* __restrict__ fb, int64_t o, int64_t r) {
  const spx_ew_params& x = p.x;
  int64_t off[SPX_MAX_IN];
#pragma unroll
  for (int j = 0; j < SPX_MAX_IN; ++j)
    if (j < x.n_in) off[j] = x.in[j].off;
  // kept dims occupy x.dims[0 .. n_kept), reduced dims x.dims[n_kept .. rank)
#pragma unroll
  for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
    if (k >= x.rank) continue;
    int64_t idx;
    if (k >= p.n_kept) {
      if (k == p.n_kept) { idx = r; } else { idx = r % x.dims[k]; r /= x.dims[k]; }
    } else {
      if (k == 0) { idx = o; } else { idx = o % x.dims[k]; o /= x.dims[k]; }
    }
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j)
      if (j < x.n_in) off[j] += idx * x.in[j].stride[k];
  }
  float in[SPX_MAX_IN];
#pragma unroll
  for (int j = 0; j < SPX_MAX_IN; ++j)
    if (j < x.n_in) in[j] = __ldg(fb + off[j]);
  float t[SPX_MAX_PROG];
#pragma unroll
  for (int i = 0; i < SPX_MAX_PROG; ++i) {
    if (i >= x.n_prog) break;
    const spx_insn ins = x.prog[i];
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int j = 0; j < SPX_MAX_IN; ++j) { if (ins.a == j) a = in[j]; if (ins.b == j) b = in[j]; }
#pragma unroll
    for (int q = 0; q < SPX_MAX_PROG; ++q) {
      if (q >= i) break;
      if (ins.a == SPX_REG_T + q) a = t[q];
      if (ins.b == SPX_REG_T + q) b = t[q];
    }
    t[i] = apply_op(ins.op, a, b, x.imm[i]);
  }
  const int reg = x.out_reg[0];
  float y = 0.f;
#pragma unroll
  for (int j = 0; j < SPX_MAX_IN; ++j) if (reg == j) y = in[j];
#pragma unroll
  for (int q = 0; q < SPX_MAX_PROG; ++q) if (reg == SPX_REG_T + q && q < x.n_prog) y = t[q];
  return y;
}

// COL mapping: block (32, 8); x -> output, y -> reduction rows.
__global__ void __launch_bounds__(256) reduce_col(const __grid_constant__ spx_reduce_params p,
                                                  int64_t chunk, int nchunks) {
  const int d = blockIdx.z;
  const float* fb = dev_ptr(p.x.base, p.x.dev_stride, d, 0);
  const int64_t o = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int c = blockIdx.y;
  const int64_t r0 = c * chunk, r1 = min(p.n_red_elems, r0 + chunk);
  float acc = ident(p.monoid);
  if (o < p.n_out)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) acc = fold(p.monoid, acc, eval_at(p, fb, o, r));
  __shared__ float sm[8][33];
  sm[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && o < p.n_out) {
    float v = sm[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < 8; ++y) v = fold(p.monoid, v, sm[y][threadIdx.x]);
    float* dst = nchunks == 1 ? dev_ptr(p.x.base, p.x.dev_stride, d, p.out_off) + o
                              : dev_ptr(p.x.base, p.x.dev_stride, d, p.scratch_off) + (int64_t)c * p.n_out + o;
    *dst = v;
  }
}

// ROW mapping: block of 8 warps; warp -> output, lanes -> reduction index.
__global__ void __launch_bounds__(256) reduce_row(const __grid_constant__ spx_reduce_params p,
                                                  int64_t chunk, int nchunks) {
  const int d = blockIdx.z;
  const float* fb = dev_ptr(p.x.base, p.x.dev_stride, d, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t o = (int64_t)blockIdx.x * 8 + warp;
  const int c = blockIdx.y;
  if (o >= p.n_out) return;
  const int64_t r0 = c * chunk, r1 = min(p.n_red_elems, r0 + chunk);
  float acc = ident(p.monoid);
  for (int64_t r = r0 + lane; r < r1; r += 32) acc = fold(p.monoid, acc, eval_at(p, fb, o, r));
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) acc = fold(p.monoid, acc, __shfl_xor_sync(0xffffffffu, acc, m));
  if (lane == 0) {
    float* dst = nchunks == 1 ? dev_ptr(p.x.base, p.x.dev_stride, d, p.out_off) + o
                              : dev_ptr(p.x.base, p.x.dev_stride, d, p.scratch_off) + (int64_t)c * p.n_out + o;
    *dst = acc;
  }
}

__global__ void reduce_final(const __grid_constant__ spx_reduce_params p, int nchunks) {
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

int spx_launch_reduce(const spx_reduce_params& p, cudaStream_t s, int* nlaunch) {
  if (p.n_out <= 0 || p.x.ndev <= 0) return 0;
  // COL when the operand's innermost (fastest) dim is a kept dim.
  const bool col = p.n_kept > 0 && p.x.rank > 0 && p.kept_stride[p.n_kept - 1] == 1;
  const int64_t per_block_out = col ? 32 : 8;
  const int64_t out_blocks = (p.n_out + per_block_out - 1) / per_block_out;
  const int64_t target = (int64_t)spx_num_sms() * 4;
  int64_t nchunks = (target + out_blocks * p.x.ndev - 1) / (out_blocks * p.x.ndev);
  const int64_t min_chunk = col ? 64 : 1024;
  const int64_t max_chunks = (p.n_red_elems + min_chunk - 1) / min_chunk;
  if (nchunks > max_chunks) nchunks = max_chunks;
  if (nchunks < 1) nchunks = 1;
  if (nchunks > 1 && p.scratch_off < 0) nchunks = 1;
  if (nchunks > 4096) nchunks = 4096;
  int64_t chunk = (p.n_red_elems + nchunks - 1) / nchunks;
  nchunks = (p.n_red_elems + chunk - 1) / chunk;
  if (nchunks < 1) nchunks = 1;
  dim3 grid((unsigned)out_blocks, (unsigned)nchunks, (unsigned)p.x.ndev);
  if (col) reduce_col<<<grid, dim3(32, 8), 0, s>>>(p, chunk, (int)nchunks);
  else reduce_row<<<grid, 256, 0, s>>>(p, chunk, (int)nchunks);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  if (nchunks > 1) {
    int64_t b = (p.n_out + 255) / 256;
    if (b > 1024) b = 1024;
    reduce_final<<<dim3((unsigned)b, (unsigned)p.x.ndev), 256, 0, s>>>(p, (int)nchunks);
    SPX_CHECK_LAUNCH();
    if (nlaunch) ++*nlaunch;
  }
  return 0;
}
