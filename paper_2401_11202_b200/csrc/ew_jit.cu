// Run-time specialised elementwise kernels (NVRTC -> sm_100a cubin).
//
// An elementwise record is one fused expression program over strided input
// views (interp.py:45-67 evaluated op by op; plan.py fuses the chain).  The
// hand-written static kernels (ew_static.cu) cover the programs the model zoo
// repeats thousands of times; everything else used to run on the register-
// machine interpreter (ew.cu), whose per-granule instruction decode, slot
// selects and runtime-divisor index math held it to 1-2 TB/s.  Here every
// other f32 record gets its own kernel, generated from the record and
// compiled by NVRTC when the plan is built:
//   * the program becomes straight-line SSA code (same IEEE operations and
//     order as the interpreter: __fadd_rn / __fmul_rn, which are never
//     contracted into FMAs, expf, NaN-propagating max), so results are
//     bit-identical to the interpreter and to the reference's numpy ops;
//   * the shape and every input's strides are compile-time constants: the
//     index decomposition is multiply-high by constants, stride-0 (broadcast)
//     dimensions vanish from the address arithmetic;
//   * float4 granules along the innermost dimension where the record allows
//     it (p.vec), two granules per thread with both granules' loads issued
//     before either's stores.
// Offsets, the arena base and the immediates stay kernel parameters, so one
// compiled kernel serves every record with the same program and geometry
// (cache keyed by the generated source and the device).  NVRTC is loaded with
// dlopen; if it is missing the record keeps the interpreter (another GPU
// kernel, never a host path) and spx_plan_record_info reports which.
#include <dlfcn.h>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>
#include <cuda.h>
#include <nvrtc.h>
#include "common.cuh"

int spx_num_sms();
bool spx_pdl_enabled();

namespace {

struct NvrtcApi {
  bool tried = false, ok = false;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) get_log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) get_cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
};

NvrtcApi& nvrtc() {
  static NvrtcApi a;
  if (a.tried) return a;
  a.tried = true;
  const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
  void* h = nullptr;
  for (const char* n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) return a;
#define SPX_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
  SPX_SYM(create, "nvrtcCreateProgram");
  SPX_SYM(compile, "nvrtcCompileProgram");
  SPX_SYM(log_size, "nvrtcGetProgramLogSize");
  SPX_SYM(get_log, "nvrtcGetProgramLog");
  SPX_SYM(cubin_size, "nvrtcGetCUBINSize");
  SPX_SYM(get_cubin, "nvrtcGetCUBIN");
  SPX_SYM(destroy, "nvrtcDestroyProgram");
#undef SPX_SYM
  a.ok = a.create && a.compile && a.log_size && a.get_log && a.cubin_size && a.get_cubin && a.destroy;
  return a;
}

template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

struct Compiled {
  std::string cubin;
  std::unordered_map<int, CUfunction> fn;      // per device ordinal
};

std::mutex g_mu;
std::unordered_map<std::string, Compiled*> g_cache;
int g_compiles = 0;

bool jit_vec(const spx_ew_params& p) { return p.vec && p.numel % 4 == 0; }

// Kernel parameter block: the generated `struct A` (8-byte aligned fields).
size_t arg_bytes(const spx_ew_params& p) {
  const int ni = p.n_in > 0 ? p.n_in : 1, np = p.n_prog > 0 ? p.n_prog : 1;
  size_t b = 16 + 8 * (size_t)ni + 8 * (size_t)p.n_out + 4 * (size_t)np;
  return (b + 7) & ~(size_t)7;
}

void fill_args(const spx_ew_params& p, std::vector<uint8_t>& buf) {
  buf.assign(arg_bytes(p), 0);
  uint8_t* q = buf.data();
  memcpy(q, &p.base, 8);
  memcpy(q + 8, &p.dev_stride, 8);
  size_t o = 16;
  const int ni = p.n_in > 0 ? p.n_in : 1;
  for (int j = 0; j < ni; ++j, o += 8) {
    const int64_t v = j < p.n_in ? p.in[j].off : 0;
    memcpy(q + o, &v, 8);
  }
  for (int j = 0; j < p.n_out; ++j, o += 8) memcpy(q + o, &p.out_off[j], 8);
  for (int i = 0; i < p.n_prog; ++i, o += 4) memcpy(q + o, &p.imm[i], 4);
}

const char* op_expr(int op, const std::string& a, const std::string& b, const std::string& im, std::string& out) {
  switch (op) {
    case SPX_OP_MOV: out = a; break;
    case SPX_OP_ADD: out = "__fadd_rn(" + a + ", " + b + ")"; break;
    case SPX_OP_MUL: out = "__fmul_rn(" + a + ", " + b + ")"; break;
    case SPX_OP_NEG: out = "-" + a; break;
    case SPX_OP_EXP: out = "expf(" + a + ")"; break;
    case SPX_OP_MAX: out = "fmx(" + a + ", " + b + ")"; break;
    case SPX_OP_IMM: out = im; break;
    case SPX_OP_ADDI: out = "__fadd_rn(" + a + ", " + im + ")"; break;
    case SPX_OP_MULI: out = "__fmul_rn(" + a + ", " + im + ")"; break;
    case SPX_OP_IADD: out = "__fadd_rn(" + im + ", " + a + ")"; break;
    case SPX_OP_IMUL: out = "__fmul_rn(" + im + ", " + a + ")"; break;
    default: return "bad opcode";
  }
  return nullptr;
}

// The scalar program of record p as a device function prog(im, x0.., y0&..).
bool gen_prog(const spx_ew_params& p, std::ostringstream& s) {
  s << "__device__ __forceinline__ float fmx(float a, float b) { return (a != a || a > b) ? a : b; }\n";
  s << "__device__ __forceinline__ void prog(const float* __restrict__ im";
  for (int j = 0; j < p.n_in; ++j) s << ", float x" << j;
  for (int o = 0; o < p.n_out; ++o) s << ", float& y" << o;
  s << ") {\n";
  for (int k = 0; k < SPX_NREG; ++k) s << "  float r" << k << " = " << (k < p.n_in ? "x" + std::to_string(k) : "0.f") << ";\n";
  for (int i = 0; i < p.n_prog; ++i) {
    const spx_insn& in = p.prog[i];
    if (in.a < 0 || in.a >= SPX_NREG || in.b < 0 || in.b >= SPX_NREG || in.dst < 0 || in.dst >= SPX_NREG) {
      spx_set_error("ew jit: slot out of range");
      return false;
    }
    std::string e;
    if (op_expr(in.op, "r" + std::to_string(in.a), "r" + std::to_string(in.b), "im[" + std::to_string(i) + "]", e)) {
      spx_set_error("ew jit: bad opcode %d", in.op);
      return false;
    }
    s << "  r" << in.dst << " = " << e << ";\n";
  }
  for (int o = 0; o < p.n_out; ++o) {
    if (p.out_reg[o] < 0 || p.out_reg[o] >= SPX_NREG) {
      spx_set_error("ew jit: output slot out of range");
      return false;
    }
    s << "  y" << o << " = r" << p.out_reg[o] << ";\n";
  }
  s << "}\n";
  return true;
}

// Loads of every input at flat element `ev` (an expression) into x<u>_<j>[W]:
// the index decomposition over the record's dims with constant divisors.
void gen_loads(const spx_ew_params& p, std::ostringstream& s, int u, const std::string& ev, bool vec, bool wide,
               bool declare = true) {
  const int W = vec ? 4 : 1;
  const int rk = p.rank > 0 ? p.rank : 1;
  const char* IX = wide ? "u64" : "u32";
  const char* SUF = wide ? "ull" : "u";
  const int64_t last = p.rank > 0 ? p.dims[rk - 1] : 1;
  if (p.n_in > 0 && declare) {
    s << "    float x" << u << "_0[" << W << "]";
    for (int j = 1; j < p.n_in; ++j) s << ", x" << u << "_" << j << "[" << W << "]";
    s << ";\n";
  }
  s << "    {\n      const " << IX << " e = " << ev << ";\n";
  bool need_outer = false;
  for (int j = 0; j < p.n_in; ++j)
    for (int k = 0; k < rk - 1; ++k)
      if (p.in[j].stride[k] != 0) need_outer = true;
  s << "      const " << IX << " c = e % " << last << SUF << ";\n";
  if (need_outer) {
    s << "      " << IX << " q = e / " << last << SUF << ";\n";
    for (int k = rk - 2; k >= 0; --k) {
      if (k == 0) s << "      const " << IX << " i0 = q;\n";
      else s << "      const " << IX << " i" << k << " = q % " << p.dims[k] << SUF << "; q /= " << p.dims[k] << SUF << ";\n";
    }
  }
  for (int j = 0; j < p.n_in; ++j) {
    s << "      const i64 o" << j << " = 0";
    for (int k = 0; k < rk - 1; ++k)
      if (p.in[j].stride[k] != 0) s << " + (i64)i" << k << " * " << p.in[j].stride[k] << "ll";
    const int64_t sl = p.rank > 0 ? p.in[j].stride[rk - 1] : 0;
    if (sl != 0) s << " + (i64)c * " << sl << "ll";
    s << ";\n";
    const std::string x = "x" + std::to_string(u) + "_" + std::to_string(j);
    if (vec && sl == 1) {
      s << "      { const float4 t = __ldg((const float4*)(p" << j << " + o" << j << ")); " << x << "[0] = t.x; " << x
        << "[1] = t.y; " << x << "[2] = t.z; " << x << "[3] = t.w; }\n";
    } else if (vec) {
      s << "      { const float t = __ldg(p" << j << " + o" << j << "); " << x << "[0] = t; " << x << "[1] = t; " << x
        << "[2] = t; " << x << "[3] = t; }\n";
    } else {
      s << "      " << x << "[0] = __ldg(p" << j << " + o" << j << ");\n";
    }
  }
  s << "    }\n";
}

// The generated CUDA source for record p (its geometry and program; offsets,
// base and immediates are parameters).  Empty + error set if unsupported.
std::string gen_source(const spx_ew_params& p) {
  const bool vec = jit_vec(p);
  const int W = vec ? 4 : 1;
  const bool wide = p.numel >= (int64_t(1) << 31);
  const char* IX = wide ? "u64" : "u32";
  const char* SUF = wide ? "ull" : "u";     // constants in the index type (32-bit divisions stay 32-bit)
  const int ni = p.n_in > 0 ? p.n_in : 1, np = p.n_prog > 0 ? p.n_prog : 1;
  std::ostringstream s;
  s << "typedef unsigned int u32; typedef unsigned long long u64; typedef long long i64;\n"
    << "struct A { u64 base; i64 dev_stride; i64 in[" << ni << "]; i64 out[" << p.n_out << "]; float imm[" << np
    << "]; };\n";
  if (!gen_prog(p, s)) return std::string();
  const int64_t n = p.numel / W;
  s << "extern \"C\" __global__ void __launch_bounds__(256) spx_ewj(const __grid_constant__ A a) {\n"
    << "  asm volatile(\"griddepcontrol.launch_dependents;\\n\\tgriddepcontrol.wait;\" ::: \"memory\");\n"
    << "  const char* b = (const char*)(a.base + (u64)((i64)blockIdx.y * a.dev_stride));\n";
  for (int j = 0; j < p.n_in; ++j) s << "  const float* __restrict__ p" << j << " = (const float*)b + a.in[" << j << "];\n";
  for (int o = 0; o < p.n_out; ++o) s << "  float* __restrict__ q" << o << " = (float*)b + a.out[" << o << "];\n";
  s << "  const " << IX << " n = " << n << SUF << ";\n"
    << "  const " << IX << " step = (" << IX << ")gridDim.x * 256u;\n";
  // granule u at index expression v: loads, then the program and the stores
  auto load = [&](int u, const char* v) {
    gen_loads(p, s, u, std::string("(") + v + ") * " + std::to_string(W) + "u", vec, wide);
  };
  auto compute = [&](int u, const char* v) {
    s << "    {\n      float y[" << p.n_out << "][" << W << "];\n";
    for (int k = 0; k < W; ++k) {
      s << "      prog(a.imm";
      for (int j = 0; j < p.n_in; ++j) s << ", x" << u << "_" << j << "[" << k << "]";
      for (int o = 0; o < p.n_out; ++o) s << ", y[" << o << "][" << k << "]";
      s << ");\n";
    }
    s << "      const " << IX << " e = (" << v << ") * " << W << "u;\n";
    for (int o = 0; o < p.n_out; ++o) {
      if (vec)
        s << "      *(float4*)(q" << o << " + e) = make_float4(y[" << o << "][0], y[" << o << "][1], y[" << o << "][2], y["
          << o << "][3]);\n";
      else
        s << "      q" << o << "[e] = y[" << o << "][0];\n";
    }
    s << "    }\n";
  };
  s << "  for (" << IX << " v = (" << IX << ")blockIdx.x * 256u + threadIdx.x; v < n; v += 2 * step) {\n"
    << "    const bool h1 = v + step < n;\n";
  load(0, "v");
  s << "    if (h1) {\n";
  load(1, "v + step");
  compute(0, "v");
  compute(1, "v + step");
  s << "    } else {\n";
  compute(0, "v");
  s << "    }\n  }\n}\n";
  return s.str();
}

// Record p with the split of its output `which` fused in (the structure of
// ew_static.cu ew_static_split_kernel): one cluster of 4 CTAs per 128 x 128
// block of the split's [rows][cols] view (32 rows per CTA, a float4 per lane
// and row), the block maximum exchanged through distributed shared memory,
// then the fp16 pieces hi = rn(x s), lo = rn(x s - hi) with s = 2^e,
// max * s in [2^14, 2^15) clamped to 2^+-60 -- bit-identical to
// split_h16_kernel.  `skip`: output `which` is read only through its pieces
// and is not stored in fp32.
std::string gen_split_source(const spx_ew_params& p, int which, bool skip) {
  const int ni = p.n_in > 0 ? p.n_in : 1, np = p.n_prog > 0 ? p.n_prog : 1;
  std::ostringstream s;
  s << "typedef unsigned int u32; typedef unsigned long long u64; typedef long long i64;\n"
    << "struct A { u64 base; i64 dev_stride; u64 dst; u64 scl; i64 sdev; i64 pitch; u64 range; i64 rows; i64 cols;"
       " i64 cb; i64 nb; i64 in[" << ni << "]; i64 out[" << p.n_out << "]; float imm[" << np << "]; };\n";
  if (!gen_prog(p, s)) return std::string();
  s << R"SRC(
__device__ __forceinline__ int sc_exp(float m) {
  const int E = (int)((__float_as_uint(m) >> 23) & 0xFF);
  const int e = (m == 0.f || E == 255) ? 0 : 141 - E;
  return e < -60 ? -60 : (e > 60 ? 60 : e);
}
__device__ __forceinline__ float pw2(int e) { return __uint_as_float((u32)(127 + e) << 23); }
__device__ __forceinline__ bool oor(float m) {
  const int E = (int)((__float_as_uint(m) >> 23) & 0xFF);
  if (m == 0.f || E == 255) return false;
  const int e = 141 - E;
  return e < -60 || e > 60;
}
__device__ __forceinline__ u32 h2(float lo, float hi) {
  u32 r; asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r;
}
__device__ __forceinline__ float hlo(u32 v) {
  float f; asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; cvt.f32.f16 %0, l; }" : "=f"(f) : "r"(v)); return f;
}
__device__ __forceinline__ float hhi(u32 v) {
  float f; asm("{ .reg .b16 l, h; mov.b32 {l, h}, %1; cvt.f32.f16 %0, h; }" : "=f"(f) : "r"(v)); return f;
}
__device__ __forceinline__ void store4(unsigned short* hi, unsigned short* lo, i64 o, const float* v, float up) {
  const float y0 = __fmul_rn(v[0], up), y1 = __fmul_rn(v[1], up), y2 = __fmul_rn(v[2], up), y3 = __fmul_rn(v[3], up);
  const u32 h01 = h2(y0, y1), h23 = h2(y2, y3);
  const u32 l01 = h2(__fsub_rn(y0, hlo(h01)), __fsub_rn(y1, hhi(h01)));
  const u32 l23 = h2(__fsub_rn(y2, hlo(h23)), __fsub_rn(y3, hhi(h23)));
  *(uint2*)(hi + o) = make_uint2(h01, h23);
  *(uint2*)(lo + o) = make_uint2(l01, l23);
}
extern "C" __global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256) spx_ewjs(const __grid_constant__ A a) {
  __shared__ float wmax[8];
  __shared__ float cmax[2][4];
  asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = blockIdx.z;
  const int crank = blockIdx.x % 4, bx = blockIdx.x / 4;
  const int cc = bx * 128 + lane * 4;
  const char* b = (const char*)(a.base + (u64)((i64)d * a.dev_stride));
)SRC";
  for (int j = 0; j < p.n_in; ++j) s << "  const float* __restrict__ p" << j << " = (const float*)b + a.in[" << j << "];\n";
  for (int o = 0; o < p.n_out; ++o) s << "  float* __restrict__ q" << o << " = (float*)b + a.out[" << o << "];\n";
  s << R"SRC(  unsigned short* hi = (unsigned short*)(a.dst + (u64)((i64)d * a.sdev));
  unsigned short* lo = hi + a.rows * a.pitch;
  const int rbs = (int)((a.rows + 127) / 128);
  const int rb0 = blockIdx.y * (int)a.nb;
  const int rb1 = rb0 + (int)a.nb < rbs ? rb0 + (int)a.nb : rbs;
)SRC";
  // the inputs of the CTA's 4 rows (32 rows / 8 warps) of one row block, kept
  // across iterations: block rb+1 is loaded while the cluster exchanges
  // block rb's maximum (as ew_static_split_kernel)
  for (int i = 0; i < 4; ++i)
    if (p.n_in > 0) {
      s << "  float x" << i << "_0[4]";
      for (int k = 1; k < p.n_in; ++k) s << ", x" << i << "_" << k << "[4]";
      s << ";\n";
    }
  s << "  auto load = [&](int rb) {\n";
  for (int i = 0; i < 4; ++i) {
    s << "   {\n    const i64 row = (i64)rb * 128 + crank * 32 + " << i * 8 << " + warp;\n"
      << "    if (row < a.rows && cc < a.cols) {\n";
    gen_loads(p, s, i, "(u32)(row * a.cols + cc)", true, false, false);
    s << "    }\n   }\n";
  }
  s << "  };\n";
  s << R"SRC(  if (rb0 < rb1) load(rb0);
  for (int rb = rb0; rb < rb1; ++rb) {
    float keep[4][4];
    float m = 0.f;
)SRC";
  for (int i = 0; i < 4; ++i) {
    s << "    {\n      const i64 row = (i64)rb * 128 + crank * 32 + " << i * 8 << " + warp;\n"
      << "      keep[" << i << "][0] = keep[" << i << "][1] = keep[" << i << "][2] = keep[" << i << "][3] = 0.f;\n"
      << "      if (row < a.rows && cc < a.cols) {\n"
      << "        float y[" << p.n_out << "][4];\n";
    for (int k = 0; k < 4; ++k) {
      s << "        prog(a.imm";
      for (int jj = 0; jj < p.n_in; ++jj) s << ", x" << i << "_" << jj << "[" << k << "]";
      for (int o = 0; o < p.n_out; ++o) s << ", y[" << o << "][" << k << "]";
      s << ");\n";
    }
    s << "        const i64 e = row * a.cols + cc;\n";
    for (int o = 0; o < p.n_out; ++o) {
      if (o == which && skip) continue;
      s << "        *(float4*)(q" << o << " + e) = make_float4(y[" << o << "][0], y[" << o << "][1], y[" << o
        << "][2], y[" << o << "][3]);\n";
    }
    s << "        for (int k = 0; k < 4; ++k) { keep[" << i << "][k] = y[" << which << "][k]; m = fmaxf(m, fabsf(keep["
      << i << "][k])); }\n      }\n    }\n";
  }
  s << R"SRC(    // block maximum over the cluster (distributed shared memory); the next
    // block's loads are issued between the barrier's arrive and its wait
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) wmax[warp] = m;
    __syncthreads();
    float* cm = cmax[rb & 1];
    if (threadIdx.x < 4) {
      float mm = wmax[0];
#pragma unroll
      for (int w = 1; w < 8; ++w) mm = fmaxf(mm, wmax[w]);
      u32 dst;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst)
                   : "r"((u32)__cvta_generic_to_shared(&cm[crank])), "r"((u32)threadIdx.x));
      asm volatile("st.shared::cluster.f32 [%0], %1;" :: "r"(dst), "f"(mm) : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    if (rb + 1 < rb1) load(rb + 1);
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    float bm = cm[0];
#pragma unroll
    for (int w = 1; w < 4; ++w) bm = fmaxf(bm, cm[w]);
    const int ex = sc_exp(bm);
    const float up = pw2(ex);
    if (threadIdx.x == 0 && crank == 0) {
      ((float*)(a.scl + (u64)((i64)d * a.sdev)))[(i64)rb * a.cb + bx] = pw2(-ex);
      if (oor(bm) && a.range) atomicAdd((u32*)a.range, 1u);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const i64 row = (i64)rb * 128 + crank * 32 + i * 8 + warp;
      if (row >= a.rows || cc >= a.cols) continue;
      store4(hi, lo, row * a.pitch + cc, keep[i], up);
    }
  }
}
)SRC";
  return s.str();
}

int compile(const std::string& src, std::string& cubin) {
  NvrtcApi& nv = nvrtc();
  if (!nv.ok) return spx_set_error("ew jit: NVRTC (libnvrtc.so.12) not loadable");
  nvrtcProgram prog;
  if (nv.create(&prog, src.c_str(), "spx_ewj.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return spx_set_error("ew jit: nvrtcCreateProgram failed");
  // nvcc's defaults otherwise (the interpreter's expf comes from the same
  // libdevice code under the same flags); the program's own adds and
  // multiplies are __fadd_rn / __fmul_rn, which are never contracted
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device"};
  const nvrtcResult r = nv.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) nv.get_log(prog, &log[0]);
    nv.destroy(&prog);
    return spx_set_error("ew jit: NVRTC compile failed: %.400s", log.c_str());
  }
  size_t n = 0;
  nv.cubin_size(prog, &n);
  cubin.assign(n, '\0');
  nv.get_cubin(prog, &cubin[0]);
  nv.destroy(&prog);
  ++g_compiles;
  return 0;
}

}  // namespace

struct SpxEwJit {
  Compiled* c = nullptr;
  std::vector<uint8_t> args;
  unsigned blocks = 1, ndev = 1;
  unsigned grid_y = 1;          // fused split: row-block groups
  bool split = false;           // spx_ewjs (fused split, 4-CTA clusters)
  size_t range_at = 0;          // fused split: byte offset of A::range (patched at first launch)
};

namespace {

Compiled* compiled_for(const std::string& src) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_cache.find(src);
  if (it != g_cache.end()) return it->second;
  Compiled* c = new Compiled();
  if (compile(src, c->cubin)) {
    delete c;
    return nullptr;
  }
  g_cache.emplace(src, c);
  return c;
}

}  // namespace

uint32_t* spx_h3_range_ew_counter();     // ew_static.cu: device address of the clamped-scale counter

// Read at every plan build (SPX_EW_JIT=0 keeps the interpreter for new plans).
bool spx_ew_jit_enabled() {
  const char* e = getenv("SPX_EW_JIT");
  return !(e && atoi(e) == 0) && nvrtc().ok;
}

// Generate + compile (cached) the kernel for record p.  Host only: no GPU needed.
int spx_ew_jit_prepare(const spx_ew_params& p, SpxEwJit** out) {
  *out = nullptr;
  if (p.dtype != SPX_DT_F32) return spx_set_error("ew jit: f32 records only");
  if (p.n_out < 1 || p.n_out > SPX_MAX_OUT || p.n_in < 0 || p.n_in > SPX_MAX_IN || p.n_prog < 0 ||
      p.n_prog > SPX_MAX_PROG || p.rank < 0 || p.rank > SPX_MAX_RANK || p.numel <= 0)
    return spx_set_error("ew jit: record outside the ABI limits");
  const std::string src = gen_source(p);
  if (src.empty()) return -1;
  Compiled* c = compiled_for(src);
  if (!c) return -1;
  SpxEwJit* j = new SpxEwJit();
  j->c = c;
  fill_args(p, j->args);
  const int64_t n = p.numel / (jit_vec(p) ? 4 : 1);
  int64_t b = (n + 511) / 512;
  const int64_t cap = (int64_t)(spx_num_sms() > 0 ? spx_num_sms() : 148) * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  j->blocks = (unsigned)b;
  j->ndev = (unsigned)p.ndev;
  *out = j;
  return 0;
}

// Record p with the split sp of its output `which` fused in (ew_static.cu
// spx_ew_split_match's conditions, plus float4 granules and < 2^31 elements).
int spx_ew_jit_split_prepare(const spx_ew_params& p, const spx_split_params& sp, int which, int skip,
                             SpxEwJit** out) {
  *out = nullptr;
  if (p.dtype != SPX_DT_F32 || !jit_vec(p) || p.numel >= (int64_t(1) << 31) || which < 0 || which >= p.n_out)
    return spx_set_error("ew jit split: record not fusable");
  const std::string src = gen_split_source(p, which, skip != 0);
  if (src.empty()) return -1;
  Compiled* c = compiled_for(src);
  if (!c) return -1;
  SpxEwJit* j = new SpxEwJit();
  j->c = c;
  j->split = true;
  const int ni = p.n_in > 0 ? p.n_in : 1, np = p.n_prog > 0 ? p.n_prog : 1;
  const size_t bytes = ((11 + ni + p.n_out) * 8 + 4 * np + 7) & ~(size_t)7;
  j->args.assign(bytes, 0);
  uint8_t* q = j->args.data();
  const uint64_t dst = sp.base + (uint64_t)(sp.dst_off * 4), scl = sp.base + (uint64_t)(sp.scl_off * 4);
  const int64_t rows = sp.rows, cols = sp.cols, cb = (sp.cols + 127) / 128, rbs = (sp.rows + 127) / 128;
  // two row blocks per cluster once the grid still covers every SM twice
  const int sms = spx_num_sms() > 0 ? spx_num_sms() : 148;
  const int64_t nb = cb * 4 * ((rbs + 1) / 2) >= 2 * sms ? 2 : 1;
  const uint64_t range = 0;
  memcpy(q + 0, &p.base, 8);
  memcpy(q + 8, &p.dev_stride, 8);
  memcpy(q + 16, &dst, 8);
  memcpy(q + 24, &scl, 8);
  memcpy(q + 32, &sp.dev_stride, 8);
  memcpy(q + 40, &sp.pitch, 8);
  memcpy(q + 48, &range, 8);
  j->range_at = 48;
  memcpy(q + 56, &rows, 8);
  memcpy(q + 64, &cols, 8);
  memcpy(q + 72, &cb, 8);
  memcpy(q + 80, &nb, 8);
  size_t o = 88;
  for (int k = 0; k < ni; ++k, o += 8) {
    const int64_t v = k < p.n_in ? p.in[k].off : 0;
    memcpy(q + o, &v, 8);
  }
  for (int k = 0; k < p.n_out; ++k, o += 8) memcpy(q + o, &p.out_off[k], 8);
  for (int k = 0; k < p.n_prog; ++k, o += 4) memcpy(q + o, &p.imm[k], 4);
  j->blocks = (unsigned)(4 * cb);
  j->grid_y = (unsigned)((rbs + nb - 1) / nb);
  j->ndev = (unsigned)p.ndev;
  *out = j;
  return 0;
}

int spx_ew_jit_launch(const SpxEwJit* j, cudaStream_t s, int* nlaunch) {
  using LoadFn = CUresult (*)(CUmodule*, const void*);
  using GetFn = CUresult (*)(CUfunction*, CUmodule, const char*);
  using LaunchFn = CUresult (*)(const CUlaunchConfig*, CUfunction, void**, void**);
  static LoadFn load = driver_fn<LoadFn>("cuModuleLoadData");
  static GetFn get = driver_fn<GetFn>("cuModuleGetFunction");
  static LaunchFn launch = driver_fn<LaunchFn>("cuLaunchKernelEx");
  if (!load || !get || !launch) return spx_set_error("ew jit: driver entry points unavailable");
  int dev = 0;
  SPX_CUDA(cudaGetDevice(&dev));
  CUfunction f = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = j->c->fn.find(dev);
    if (it != j->c->fn.end()) {
      f = it->second;
    } else {
      CUmodule m;
      CUresult r = load(&m, j->c->cubin.data());
      if (r != CUDA_SUCCESS) return spx_set_error("ew jit: cuModuleLoadData failed (%d)", (int)r);
      r = get(&f, m, j->split ? "spx_ewjs" : "spx_ewj");
      if (r != CUDA_SUCCESS) return spx_set_error("ew jit: cuModuleGetFunction failed (%d)", (int)r);
      j->c->fn.emplace(dev, f);
    }
  }
  if (j->split) {
    uint64_t have = 0;
    memcpy(&have, j->args.data() + j->range_at, 8);
    if (!have) {
      const uint64_t r = reinterpret_cast<uint64_t>(spx_h3_range_ew_counter());
      memcpy(const_cast<uint8_t*>(j->args.data()) + j->range_at, &r, 8);
    }
  }
  CUlaunchConfig cfg = {};
  cfg.gridDimX = j->blocks;
  cfg.gridDimY = j->split ? j->grid_y : j->ndev;
  cfg.gridDimZ = j->split ? j->ndev : 1;
  cfg.blockDimX = 256;
  cfg.blockDimY = 1;
  cfg.blockDimZ = 1;
  cfg.hStream = reinterpret_cast<CUstream>(s);
  CUlaunchAttribute at[1];
  if (spx_pdl_enabled()) {
    at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    at[0].value.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  void* params[1] = {const_cast<uint8_t*>(j->args.data())};
  const CUresult r = launch(&cfg, f, params, nullptr);
  if (r != CUDA_SUCCESS) return spx_set_error("ew jit: cuLaunchKernelEx failed (%d)", (int)r);
  if (nlaunch) ++*nlaunch;
  return 0;
}

void spx_ew_jit_free(SpxEwJit* j) { delete j; }

// ---- C-ABI (tests, tools) ----
extern "C" {

int spx_ew_jit_available(void) { return nvrtc().ok ? 1 : 0; }

int spx_ew_jit_source(const spx_ew_params* p, char* buf, int64_t cap) {
  const std::string s = gen_source(*p);
  if (s.empty()) return -1;
  if ((int64_t)s.size() + 1 > cap) return spx_set_error("ew jit: source needs %zu bytes", s.size() + 1);
  memcpy(buf, s.c_str(), s.size() + 1);
  return (int)s.size();
}

int spx_ew_jit_compile(const spx_ew_params* p) {
  SpxEwJit* j = nullptr;
  if (spx_ew_jit_prepare(*p, &j)) return -1;
  spx_ew_jit_free(j);
  return 0;
}

int spx_ew_jit_split_source(const spx_ew_params* p, int which, int skip, char* buf, int64_t cap) {
  const std::string s = gen_split_source(*p, which, skip != 0);
  if (s.empty()) return -1;
  if ((int64_t)s.size() + 1 > cap) return spx_set_error("ew jit: source needs %zu bytes", s.size() + 1);
  memcpy(buf, s.c_str(), s.size() + 1);
  return (int)s.size();
}

int spx_ew_jit_split_compile(const spx_ew_params* p, const spx_split_params* sp, int which, int skip) {
  SpxEwJit* j = nullptr;
  if (spx_ew_jit_split_prepare(*p, *sp, which, skip, &j)) return -1;
  spx_ew_jit_free(j);
  return 0;
}

int spx_ew_jit_stats(int* compiles, int* cached) {
  std::lock_guard<std::mutex> lk(g_mu);
  *compiles = g_compiles;
  *cached = (int)g_cache.size();
  return 0;
}

}  // extern "C"
