// int32 arithmetic (the IR's second element kind, ir.py:14): when every input
// of a call is int32 the reference computes in int32 (np.result_type,
// spmd_interp.py:173; constants adopt it, interp.py:39-41) with numpy's
// wrapping ufuncs.  Data movement (views, all_slice/all_gather/all_to_all) is
// type-agnostic and shares the f32 kernels; these are the arithmetic records:
//   elementwise programs  add / mul / neg (/ max), modulo 2^32
//   reduce max            (np.max keeps int32; np.sum would widen to int64 and
//                          is refused by the compiler)
//   all_reduce / reduce_scatter  left fold in group order (np.add / np.maximum)
//   matmul                int32 products summed modulo 2^32 (numpy's integer
//                          matmul) -- order-independent, so any schedule is
//                          bit-exact.
// Not a hot path: plain SIMT kernels, one element (or output) per thread.
#include "common.cuh"

namespace {

SPX_DEV int32_t i_add(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
SPX_DEV int32_t i_mul(int32_t a, int32_t b) { return (int32_t)((uint32_t)a * (uint32_t)b); }
SPX_DEV int32_t i_neg(int32_t a) { return (int32_t)(0u - (uint32_t)a); }
SPX_DEV int32_t i_max(int32_t a, int32_t b) { return a > b ? a : b; }

SPX_DEV int32_t i_op(int op, int32_t a, int32_t b, int32_t c) {
  switch (op) {
    case SPX_OP_MOV: return a;
    case SPX_OP_ADD: return i_add(a, b);
    case SPX_OP_MUL: return i_mul(a, b);
    case SPX_OP_NEG: return i_neg(a);
    case SPX_OP_MAX: return i_max(a, b);
    case SPX_OP_IMM: return c;
    case SPX_OP_ADDI: return i_add(a, c);
    case SPX_OP_MULI: return i_mul(a, c);
    case SPX_OP_IADD: return i_add(c, a);
    case SPX_OP_IMUL: return i_mul(c, a);
  }
  return 0;
}

SPX_DEV int32_t* iptr(uint64_t base, int64_t dev_stride, int d, int64_t off) {
  return reinterpret_cast<int32_t*>(base + (uint64_t)((int64_t)d * dev_stride) + (uint64_t)(off * 4));
}

// value of the expression program at logical element e of p.dims (outputs:
// every slot; the caller picks out_reg)
SPX_DEV void i_eval(const spx_ew_params& p, const int32_t* fb, int64_t e, int32_t (&r)[SPX_NREG]) {
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
#pragma unroll
  for (int j = 0; j < SPX_MAX_IN; ++j)
    if (j < p.n_in) r[j] = fb[off[j]];
#pragma unroll 1
  for (int i = 0; i < p.n_prog; ++i) {
    const spx_insn in = p.prog[i];
    const int32_t c = __float_as_int(p.imm[i]);
    int32_t a = 0, b = 0;
#pragma unroll
    for (int k = 0; k < SPX_NREG; ++k) {
      if (k == in.a) a = r[k];
      if (k == in.b) b = r[k];
    }
    const int32_t y = i_op(in.op, a, b, c);
#pragma unroll
    for (int k = 0; k < SPX_NREG; ++k)
      if (k == in.dst) r[k] = y;
  }
}

SPX_DEV int32_t pick(const int32_t (&r)[SPX_NREG], int k) {
  int32_t v = 0;
#pragma unroll
  for (int i = 0; i < SPX_NREG; ++i)
    if (i == k) v = r[i];
  return v;
}

__global__ void __launch_bounds__(256) ew_i32_kernel(const __grid_constant__ spx_ew_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const int32_t* fb = iptr(p.base, p.dev_stride, d, 0);
  int32_t* ob = iptr(p.base, p.dev_stride, d, 0);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.numel;
       e += (int64_t)gridDim.x * blockDim.x) {
    int32_t r[SPX_NREG];
    i_eval(p, fb, e, r);
#pragma unroll
    for (int o = 0; o < SPX_MAX_OUT; ++o)
      if (o < p.n_out) ob[p.out_off[o] + e] = pick(r, p.out_reg[o]);
  }
}

// one thread per output: x.dims = kept dims ++ reduced dims (row-major)
__global__ void __launch_bounds__(256) reduce_max_i32_kernel(const __grid_constant__ spx_reduce_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const int32_t* fb = iptr(p.x.base, p.x.dev_stride, d, 0);
  int32_t* ob = iptr(p.x.base, p.x.dev_stride, d, p.out_off);
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < p.n_out;
       o += (int64_t)gridDim.x * blockDim.x) {
    int32_t acc = 0;
    for (int64_t k = 0; k < p.n_red_elems; ++k) {
      int32_t r[SPX_NREG];
      i_eval(p.x, fb, o * p.n_red_elems + k, r);
      const int32_t v = pick(r, p.x.out_reg[0]);
      acc = k == 0 ? v : i_max(acc, v);
    }
    ob[o] = acc;
  }
}

__global__ void __launch_bounds__(256) creduce_i32_kernel(const __grid_constant__ spx_creduce_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.y;
  const int32_t* const* src = reinterpret_cast<const int32_t* const*>(p.src);
  const int32_t* mem = reinterpret_cast<const int32_t*>(p.members) + (int64_t)d * p.n_members;
  const int64_t b = reinterpret_cast<const int64_t*>(p.base_off)[d];
  int32_t* out = reinterpret_cast<int32_t* const*>(p.dst)[d];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.numel;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = e, soff = b;
#pragma unroll
    for (int k = SPX_MAX_RANK - 1; k >= 0; --k) {
      if (k >= p.rank) continue;
      const int64_t lk = (k == 0) ? rem : rem % p.dims[k];
      rem = (k == 0) ? 0 : rem / p.dims[k];
      soff += lk * p.sstride[k];
    }
    int32_t acc = src[mem[0]][soff];
    for (int j = 1; j < p.n_members; ++j) {
      const int32_t v = src[mem[j]][soff];
      acc = p.monoid == 0 ? i_add(acc, v) : i_max(acc, v);
    }
    out[e] = acc;
  }
}

// C[m][n] = sum_k A[m][k] * B[k][n] mod 2^32; 16x16 threads, one output each
__global__ void __launch_bounds__(256) gemm_i32_kernel(const __grid_constant__ spx_gemm_params p) {
  SPX_PDL_ENTRY();
  const int d = blockIdx.z;
  const int32_t* A = iptr(p.base, p.dev_stride, d, p.a_off);
  const int32_t* B = iptr(p.base, p.dev_stride, d, p.b_off);
  int32_t* C = iptr(p.base, p.dev_stride, d, p.c_off);
  const int64_t sam = p.a_mn_major ? 1 : p.lda, sak = p.a_mn_major ? p.lda : 1;
  const int64_t sbk = p.b_k_major ? 1 : p.ldb, sbn = p.b_k_major ? p.ldb : 1;
  const int m = blockIdx.y * 16 + threadIdx.y, n = blockIdx.x * 16 + threadIdx.x;
  if (m >= p.M || n >= p.N) return;
  uint32_t acc = 0;
  for (int k = 0; k < p.K; ++k) acc += (uint32_t)A[m * sam + k * sak] * (uint32_t)B[k * sbk + n * sbn];
  C[(int64_t)m * p.ldc + n] = (int32_t)acc;
}

unsigned grid1(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)spx_num_sms() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

int spx_launch_ew_i32(const spx_ew_params& p, cudaStream_t s, int* nlaunch) {
  if (p.numel <= 0 || p.ndev <= 0) return 0;
  if (p.n_prog > SPX_MAX_PROG || p.n_in > SPX_MAX_IN || p.n_out > SPX_MAX_OUT)
    return spx_set_error("ew i32: program exceeds ABI limits");
  for (int i = 0; i < p.n_prog; ++i)
    if (p.prog[i].op == SPX_OP_EXP) return spx_set_error("ew i32: exp has no int32 result (numpy widens to float64)");
  spx_launch(ew_i32_kernel, dim3(grid1(p.numel), (unsigned)p.ndev), 256, 0, s, p);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

int spx_launch_reduce_i32(const spx_reduce_params& p, cudaStream_t s, int* nlaunch) {
  if (p.monoid != 1) return spx_set_error("reduce i32: only max keeps int32 (np.sum widens to int64)");
  if (p.n_out <= 0) return 0;
  spx_launch(reduce_max_i32_kernel, dim3(grid1(p.n_out), (unsigned)p.x.ndev), 256, 0, s, p);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

int spx_launch_creduce_i32(const spx_creduce_params& p, cudaStream_t s, int* nlaunch) {
  if (p.numel <= 0) return 0;
  spx_launch(creduce_i32_kernel, dim3(grid1(p.numel), (unsigned)p.ndev), 256, 0, s, p);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

int spx_launch_gemm_i32(const spx_gemm_params& p, cudaStream_t s, int* nlaunch) {
  if (p.M <= 0 || p.N <= 0) return 0;
  spx_launch(gemm_i32_kernel, dim3((p.N + 15) / 16, (p.M + 15) / 16, p.ndev), dim3(16, 16), 0, s, p);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}
