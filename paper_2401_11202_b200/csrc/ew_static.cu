// Compile-time-specialised fused elementwise kernels for the programs the
// reference's model zoo actually produces (models.py:43-85: momentum update,
// square activation and its gradient, residual add, scale, sub).  The plan
// still emits the generic register-machine program (ew.cu); spx_plan_add
// matches it against this catalog and, on a hit, launches straight-line code
// with the same per-op IEEE rounding (bit-identical results) but no
// interpretation overhead -- ncu showed the interpreter latency-bound at
// 0.9-1.7 TB/s on exactly these programs.
#include <cstdlib>
#include "interp.cuh"
#include "h3_split.cuh"

__device__ uint32_t g_h3_range_ew = 0;   // fused splits whose block scale was clamped

namespace {

constexpr uint32_t ins(int op, int a, int b, int d) {
  return (uint32_t)op | ((uint32_t)a << 8) | ((uint32_t)b << 16) | ((uint32_t)d << 24);
}

template <uint32_t I>
SPX_DEV void step(Vec<4>* r, float c) {
  constexpr int op = I & 255, a = (I >> 8) & 255, b = (I >> 16) & 255, d = (I >> 24) & 255;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float x = r[a].v[k], y = r[b].v[k];
    float z;
    if (op == SPX_OP_ADD) z = f_add(x, y);
    else if (op == SPX_OP_MUL) z = f_mul(x, y);
    else if (op == SPX_OP_NEG) z = -x;
    else if (op == SPX_OP_EXP) z = expf(x);
    else if (op == SPX_OP_MAX) z = f_max(x, y);
    else if (op == SPX_OP_IMM) z = c;
    else if (op == SPX_OP_ADDI) z = f_add(x, c);
    else if (op == SPX_OP_MULI) z = f_mul(x, c);
    else if (op == SPX_OP_IADD) z = f_add(c, x);
    else if (op == SPX_OP_IMUL) z = f_mul(c, x);
    else z = x;
    r[d].v[k] = z;
  }
}

template <uint32_t... I, int... Ix>
SPX_DEV void run_static(Vec<4>* r, const float* imm, std::integer_sequence<int, Ix...>) {
  (step<I>(r, imm[Ix]), ...);
}

// NIN inputs, NOUT outputs (slots O0, O1), program I...; 2 float4 granules per
// thread per iteration with all loads hoisted.
template <int NIN, int NOUT, int O0, int O1, uint32_t... I>
__global__ void __launch_bounds__(256) ew_static_kernel(const __grid_constant__ spx_ew_params p) {
  SPX_PDL_ENTRY();
  constexpr int U = 2;
  const int d = blockIdx.y;
  const float* __restrict__ fb = dev_ptr(p.base, p.dev_stride, d, 0);
  float* __restrict__ ob = dev_ptr(p.base, p.dev_stride, d, 0);
  const uint32_t nvec = (uint32_t)(p.numel >> 2);
  const bool two_d = p.rank == 2;
  const uint32_t cols = (uint32_t)(two_d ? p.dims[1] : p.numel);
  const uint32_t step_ = gridDim.x * blockDim.x;
  float* out0 = ob + p.out_off[0];
  float* out1 = ob + p.out_off[NOUT > 1 ? 1 : 0];
  for (uint32_t v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < nvec; v0 += step_ * U) {
    Vec<4> r[U][SPX_NREG];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t v = v0 + u * step_;
      if (v >= nvec) break;
      const uint32_t e = v << 2;
      const uint32_t row = two_d ? e / cols : 0u;
      const uint32_t col = e - row * cols;
#pragma unroll
      for (int j = 0; j < NIN; ++j) {
        const float* src = fb + p.in[j].off + (two_d ? (size_t)row * p.in[j].stride[0] : 0);
        if (p.in[j].stride[p.rank - 1] != 0) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(src + col));
          r[u][j].v[0] = t.x; r[u][j].v[1] = t.y; r[u][j].v[2] = t.z; r[u][j].v[3] = t.w;
        } else {
          const float t = __ldg(src);
          r[u][j].v[0] = t; r[u][j].v[1] = t; r[u][j].v[2] = t; r[u][j].v[3] = t;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t v = v0 + u * step_;
      if (v >= nvec) break;
      run_static<I...>(r[u], p.imm, std::make_integer_sequence<int, (int)sizeof...(I)>{});
      const size_t e = (size_t)v << 2;
      *reinterpret_cast<float4*>(out0 + e) = make_float4(r[u][O0].v[0], r[u][O0].v[1], r[u][O0].v[2], r[u][O0].v[3]);
      if (NOUT > 1)
        *reinterpret_cast<float4*>(out1 + e) =
            make_float4(r[u][O1].v[0], r[u][O1].v[1], r[u][O1].v[2], r[u][O1].v[3]);
    }
  }
}

// Pieces of output `which` for the block-scaled 3xFP16 GEMM (h3_split.cuh):
// the output viewed as [rows][cols] row-major, pieces [2][rows][pitch] fp16.
struct EwSplit {
  uint64_t dst, scl;        // device-0 addresses
  int64_t dev_stride, pitch;
  int rows, cols, cb, which;
  int nb;                   // row blocks per cluster (pipelined)
  int skip;                 // 1: output `which` is read only through its pieces -- no fp32 store
};

// The same program over 128 x 128 output blocks, a cluster of H3_CL CTAs per
// block (32 rows each): outputs are stored as usual, and the block maximum of
// output `which` (exchanged through distributed shared memory) gives the
// scale for its fp16 pieces -- the split the GEMMs reading this output need,
// without reading it back from HBM.
template <int NIN, int NOUT, int O0, int O1, uint32_t... I>
__global__ void __cluster_dims__(H3_CL, 1, 1) __launch_bounds__(256)
ew_static_split_kernel(const __grid_constant__ spx_ew_params p, const __grid_constant__ EwSplit q) {
  __shared__ float wmax[8];
  __shared__ float cmax[2][H3_CL];
  SPX_PDL_ENTRY();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = blockIdx.z;
  const int crank = blockIdx.x % H3_CL, bx = blockIdx.x / H3_CL;
  const int c = bx * H3_BLOCK + lane * 4;
  const float* __restrict__ fb = dev_ptr(p.base, p.dev_stride, d, 0);
  float* __restrict__ ob = dev_ptr(p.base, p.dev_stride, d, 0);
  const bool two_d = p.rank == 2;
  const int64_t ecols = two_d ? p.dims[1] : p.numel;
  float* out0 = ob + p.out_off[0];
  float* out1 = ob + p.out_off[NOUT > 1 ? 1 : 0];
  __half* hi = reinterpret_cast<__half*>(q.dst + (uint64_t)((int64_t)d * q.dev_stride));
  __half* lo = hi + (int64_t)q.rows * q.pitch;
  // q.nb row blocks per cluster, software-pipelined: the inputs of block
  // it + 1 are loaded before the pieces of block it are stored, so the read
  // and write streams of consecutive blocks overlap
  auto load = [&](int rb, Vec<4> (&r)[H3_V][SPX_NREG]) {
#pragma unroll
    for (int i = 0; i < H3_V; ++i) {
      const int row = rb * H3_BLOCK + crank * H3_ROWS + i * 8 + warp;
      if (row >= q.rows || c >= q.cols) continue;
      const int64_t e = (int64_t)row * q.cols + c;
      const int64_t erow = two_d ? e / ecols : 0;
      const int64_t ecol = e - erow * ecols;
#pragma unroll
      for (int j = 0; j < NIN; ++j) {
        const float* src = fb + p.in[j].off + (two_d ? erow * p.in[j].stride[0] : 0);
        if (p.in[j].stride[p.rank - 1] != 0) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(src + ecol));
          r[i][j].v[0] = t.x; r[i][j].v[1] = t.y; r[i][j].v[2] = t.z; r[i][j].v[3] = t.w;
        } else {
          const float t = __ldg(src);
          r[i][j].v[0] = t; r[i][j].v[1] = t; r[i][j].v[2] = t; r[i][j].v[3] = t;
        }
      }
    }
  };
  const int rb0 = blockIdx.y * q.nb;
  const int rb1 = min(rb0 + q.nb, (q.rows + H3_BLOCK - 1) / H3_BLOCK);
  Vec<4> r[H3_V][SPX_NREG];
  load(rb0, r);
  for (int rb = rb0; rb < rb1; ++rb) {
    float4 keep[H3_V];
    float4 other[H3_V];     // the output that is not split (NOUT == 2)
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < H3_V; ++i) {
      const int row = rb * H3_BLOCK + crank * H3_ROWS + i * 8 + warp;
      keep[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      other[i] = keep[i];
      if (row >= q.rows || c >= q.cols) continue;
      run_static<I...>(r[i], p.imm, std::make_integer_sequence<int, (int)sizeof...(I)>{});
      const float4 y0 = make_float4(r[i][O0].v[0], r[i][O0].v[1], r[i][O0].v[2], r[i][O0].v[3]);
      if (NOUT > 1) {
        const float4 y1 = make_float4(r[i][O1].v[0], r[i][O1].v[1], r[i][O1].v[2], r[i][O1].v[3]);
        keep[i] = q.which ? y1 : y0;
        other[i] = q.which ? y0 : y1;
      } else {
        keep[i] = y0;
      }
      m = h3_absmax4(m, keep[i]);
    }
    // publish the partial maximum first, THEN issue the fp32 output stores and
    // the next block's loads: the cluster barrier's release does not wait for them
    h3_cluster_max_arrive(m, wmax, cmax[rb & 1], crank);
#pragma unroll
    for (int i = 0; i < H3_V; ++i) {
      const int row = rb * H3_BLOCK + crank * H3_ROWS + i * 8 + warp;
      if (row >= q.rows || c >= q.cols) continue;
      const int64_t e = (int64_t)row * q.cols + c;
      float* ok = q.which ? out1 : out0;       // the split output
      float* oo = q.which ? out0 : out1;
      if (!q.skip) *reinterpret_cast<float4*>(ok + e) = keep[i];
      if (NOUT > 1) *reinterpret_cast<float4*>(oo + e) = other[i];
    }
    if (rb + 1 < rb1) load(rb + 1, r);
    m = h3_cluster_max_wait(cmax[rb & 1]);
    const int ex = h3_scale_exp(m);
    const float up = h3_pow2(ex);
    if (threadIdx.x == 0 && crank == 0) {
      reinterpret_cast<float*>(q.scl + (uint64_t)((int64_t)d * q.dev_stride))[rb * q.cb + bx] = h3_pow2(-ex);
      if (h3_out_of_range(m)) atomicAdd(&g_h3_range_ew, 1u);
    }
#pragma unroll
    for (int i = 0; i < H3_V; ++i) {
      const int row = rb * H3_BLOCK + crank * H3_ROWS + i * 8 + warp;
      if (row >= q.rows || c >= q.cols) continue;
      h3_store4(hi, lo, (int64_t)row * q.pitch + c, keep[i], up, 4);
    }
  }
}

struct Entry {
  int n_in, n_out, out0, out1, n_prog;
  uint32_t prog[8];
  void (*launch)(const spx_ew_params&, dim3, cudaStream_t);
  void (*launch_split)(const spx_ew_params&, const EwSplit&, dim3, cudaStream_t);
};

template <int NIN, int NOUT, int O0, int O1, uint32_t... I>
void launch_static(const spx_ew_params& p, dim3 g, cudaStream_t s) {
  spx_launch(ew_static_kernel<NIN, NOUT, O0, O1, I...>, g, 256, 0, s, p);
}

template <int NIN, int NOUT, int O0, int O1, uint32_t... I>
void launch_static_split(const spx_ew_params& p, const EwSplit& q, dim3 g, cudaStream_t s) {
  spx_launch(ew_static_split_kernel<NIN, NOUT, O0, O1, I...>, g, 256, 0, s, p, q);
}

#define OP(x) SPX_OP_##x
// The catalog (program slots as allocated by plan.Program.build).
#define E(NIN, NOUT, O0, O1, N, ...) \
  {NIN, NOUT, O0, O1, N, {__VA_ARGS__}, launch_static<NIN, NOUT, O0, O1, __VA_ARGS__>, \
   launch_static_split<NIN, NOUT, O0, O1, __VA_ARGS__>}
const Entry kCatalog[] = {
    // momentum update  m' = c0*m + g ; p' = p + -(c2*m')        (models.py:79-85)
    E(3, 2, 0, 1, 5, ins(OP(IMUL), 0, 0, 0), ins(OP(ADD), 0, 1, 0), ins(OP(IMUL), 0, 0, 1), ins(OP(NEG), 1, 0, 1),
      ins(OP(ADD), 2, 1, 1)),
    // square-activation gradient  dh * (c*z)                    (models.py:76-77)
    E(2, 1, 0, 0, 2, ins(OP(IMUL), 1, 0, 1), ins(OP(MUL), 0, 1, 0)),
    // residual / bias add
    E(2, 1, 0, 0, 1, ins(OP(ADD), 0, 1, 0)),
    // square activation  z * z                                   (models.py:73-74)
    E(1, 1, 0, 0, 1, ins(OP(MUL), 0, 0, 0)),
    // scale  c * x
    E(1, 1, 0, 0, 1, ins(OP(IMUL), 0, 0, 0)),
    // sub  a + -b  (+ c)
    E(3, 1, 0, 0, 3, ins(OP(ADD), 0, 1, 0), ins(OP(NEG), 2, 0, 1), ins(OP(ADD), 0, 1, 0)),
    E(2, 1, 0, 0, 2, ins(OP(NEG), 1, 0, 1), ins(OP(ADD), 0, 1, 0)),
    // product
    E(2, 1, 0, 0, 1, ins(OP(MUL), 0, 1, 0)),
};
#undef E
#undef OP

}  // namespace

// Catalog index for a program, or -1.  Also requires the vector-path layout.
int spx_ew_static_match(const spx_ew_params& p) {
  if (p.dtype != SPX_DT_F32 || !p.vec || p.numel % 4 || p.rank > 2 || p.numel >= (int64_t(1) << 31)) return -1;
  for (int i = 0; i < (int)(sizeof(kCatalog) / sizeof(kCatalog[0])); ++i) {
    const Entry& c = kCatalog[i];
    if (c.n_in != p.n_in || c.n_out != p.n_out || c.n_prog != p.n_prog) continue;
    if (p.out_reg[0] != c.out0 || (c.n_out > 1 && p.out_reg[1] != c.out1)) continue;
    bool ok = true;
    for (int k = 0; k < c.n_prog && ok; ++k) {
      const spx_insn& q = p.prog[k];
      const uint32_t want = c.prog[k];
      const int op = want & 255, a = (want >> 8) & 255, b = (want >> 16) & 255, d = (want >> 24) & 255;
      const bool unary = op == SPX_OP_NEG || op == SPX_OP_EXP || op == SPX_OP_IMM || op >= SPX_OP_ADDI;
      ok = q.op == op && q.a == a && q.dst == d && (unary || q.b == b);
    }
    if (ok) return i;
  }
  return -1;
}

int spx_launch_ew_static(int id, const spx_ew_params& p, cudaStream_t s, int* nlaunch) {
  const int64_t nv = p.numel / 4;
  int64_t b = (nv / 2 + 255) / 256;
  const int64_t cap = (int64_t)spx_num_sms() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  kCatalog[id].launch(p, dim3((unsigned)b, (unsigned)p.ndev), s);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}

uint32_t* spx_h3_range_ew_counter() {
  void* a = nullptr;
  if (cudaGetSymbolAddress(&a, g_h3_range_ew) != cudaSuccess) return nullptr;
  return static_cast<uint32_t*>(a);
}

int spx_h3_range_ew(uint32_t* out, int reset) {
  SPX_CUDA(cudaMemcpyFromSymbol(out, g_h3_range_ew, sizeof(uint32_t)));
  if (reset && *out) {
    const uint32_t z = 0;
    SPX_CUDA(cudaMemcpyToSymbol(g_h3_range_ew, &z, sizeof(z)));
  }
  return 0;
}

// Can split record `sp` be fused into static elementwise record `p`?  Returns
// the output index it splits, or -1.
int spx_ew_split_match(const spx_ew_params& p, const spx_split_params& sp) {
  if (!p.vec || sp.ld != sp.cols || (int64_t)sp.rows * sp.cols != p.numel || sp.cols % 4 || sp.ndev != p.ndev ||
      sp.base != p.base || sp.dev_stride != p.dev_stride)
    return -1;
  for (int j = 0; j < p.n_out; ++j)
    if (p.out_off[j] == sp.src_off) return j;
  return -1;
}

int spx_launch_ew_static_split(int id, const spx_ew_params& p, const spx_split_params& sp, int which,
                               cudaStream_t s, int* nlaunch) {
  EwSplit q;
  q.dst = sp.base + (uint64_t)(sp.dst_off * 4);
  q.scl = sp.base + (uint64_t)(sp.scl_off * 4);
  q.dev_stride = sp.dev_stride;
  q.pitch = sp.pitch;
  q.rows = sp.rows;
  q.cols = sp.cols;
  q.cb = (sp.cols + H3_BLOCK - 1) / H3_BLOCK;
  q.which = which;
  static int po = -1;
  if (po < 0) {
    const char* e = getenv("SPX_PIECES_ONLY");
    po = e ? atoi(e) != 0 : 1;
  }
  q.skip = po && (sp.flags & SPX_SPLIT_PIECES_ONLY) ? 1 : 0;
  const int rbs = (sp.rows + H3_BLOCK - 1) / H3_BLOCK;
  // two row blocks per cluster once the grid still covers every SM twice
  static int nbe = -1;
  if (nbe < 0) {
    const char* e = getenv("SPX_EW_SPLIT_NB");
    nbe = e ? atoi(e) : 0;
  }
  q.nb = nbe > 0 ? nbe : ((int64_t)q.cb * H3_CL * ((rbs + 1) / 2) >= 2 * spx_num_sms() ? 2 : 1);
  const dim3 g((unsigned)(H3_CL * q.cb), (unsigned)((rbs + q.nb - 1) / q.nb), (unsigned)p.ndev);
  kCatalog[id].launch_split(p, q, g, s);
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}
