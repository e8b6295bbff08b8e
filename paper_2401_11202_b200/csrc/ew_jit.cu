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

// The generated CUDA source for record p (its geometry and program; offsets,
// base and immediates are parameters).  Empty + error set if unsupported.
std::string gen_source(const spx_ew_params& p) {
  const bool vec = jit_vec(p);
  const int W = vec ? 4 : 1;
  const int rk = p.rank > 0 ? p.rank : 1;
  const bool wide = p.numel >= (int64_t(1) << 31);
  const char* IX = wide ? "u64" : "u32";
  const char* SUF = wide ? "ull" : "u";     // constants in the index type (32-bit divisions stay 32-bit)
  const int ni = p.n_in > 0 ? p.n_in : 1, np = p.n_prog > 0 ? p.n_prog : 1;
  std::ostringstream s;
  s << "typedef unsigned int u32; typedef unsigned long long u64; typedef long long i64;\n"
    << "struct A { u64 base; i64 dev_stride; i64 in[" << ni << "]; i64 out[" << p.n_out << "]; float imm[" << np
    << "]; };\n"
    << "__device__ __forceinline__ float fmx(float a, float b) { return (a != a || a > b) ? a : b; }\n";
  // the program, one scalar lane
  s << "__device__ __forceinline__ void prog(const float* __restrict__ im";
  for (int j = 0; j < p.n_in; ++j) s << ", float x" << j;
  for (int o = 0; o < p.n_out; ++o) s << ", float& y" << o;
  s << ") {\n";
  for (int k = 0; k < SPX_NREG; ++k) s << "  float r" << k << " = " << (k < p.n_in ? "x" + std::to_string(k) : "0.f") << ";\n";
  for (int i = 0; i < p.n_prog; ++i) {
    const spx_insn& in = p.prog[i];
    if (in.a < 0 || in.a >= SPX_NREG || in.b < 0 || in.b >= SPX_NREG || in.dst < 0 || in.dst >= SPX_NREG) {
      spx_set_error("ew jit: slot out of range");
      return std::string();
    }
    std::string e;
    if (op_expr(in.op, "r" + std::to_string(in.a), "r" + std::to_string(in.b), "im[" + std::to_string(i) + "]", e)) {
      spx_set_error("ew jit: bad opcode %d", in.op);
      return std::string();
    }
    s << "  r" << in.dst << " = " << e << ";\n";
  }
  for (int o = 0; o < p.n_out; ++o) {
    if (p.out_reg[o] < 0 || p.out_reg[o] >= SPX_NREG) {
      spx_set_error("ew jit: output slot out of range");
      return std::string();
    }
    s << "  y" << o << " = r" << p.out_reg[o] << ";\n";
  }
  s << "}\n";
  // the kernel
  const int64_t last = p.rank > 0 ? p.dims[rk - 1] : 1;
  const int64_t n = p.numel / W;
  s << "extern \"C\" __global__ void __launch_bounds__(256) spx_ewj(const __grid_constant__ A a) {\n"
    << "  asm volatile(\"griddepcontrol.launch_dependents;\\n\\tgriddepcontrol.wait;\" ::: \"memory\");\n"
    << "  const char* b = (const char*)(a.base + (u64)((i64)blockIdx.y * a.dev_stride));\n";
  for (int j = 0; j < p.n_in; ++j) s << "  const float* __restrict__ p" << j << " = (const float*)b + a.in[" << j << "];\n";
  for (int o = 0; o < p.n_out; ++o) s << "  float* __restrict__ q" << o << " = (float*)b + a.out[" << o << "];\n";
  s << "  const " << IX << " n = " << n << SUF << ";\n"
    << "  const " << IX << " step = (" << IX << ")gridDim.x * 256u;\n";
  // granule loads: x<u>_<j>[W]
  auto load = [&](int u, const char* v) {
    if (p.n_in > 0) {
      s << "    float x" << u << "_0[" << W << "]";
      for (int j = 1; j < p.n_in; ++j) s << ", x" << u << "_" << j << "[" << W << "]";
      s << ";\n";
    }
    s << "    {\n      const " << IX << " e = (" << v << ") * " << W << "u;\n";
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
      if (vec && sl == 1) {
        s << "      { const float4 t = __ldg((const float4*)(p" << j << " + o" << j << ")); x" << u << "_" << j
          << "[0] = t.x; x" << u << "_" << j << "[1] = t.y; x" << u << "_" << j << "[2] = t.z; x" << u << "_" << j
          << "[3] = t.w; }\n";
      } else if (vec) {
        s << "      { const float t = __ldg(p" << j << " + o" << j << "); x" << u << "_" << j << "[0] = t; x" << u << "_"
          << j << "[1] = t; x" << u << "_" << j << "[2] = t; x" << u << "_" << j << "[3] = t; }\n";
      } else {
        s << "      x" << u << "_" << j << "[0] = __ldg(p" << j << " + o" << j << ");\n";
      }
    }
    s << "    }\n";
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
};

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
  Compiled* c = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(src);
    if (it != g_cache.end()) {
      c = it->second;
    } else {
      c = new Compiled();
      if (compile(src, c->cubin)) {
        delete c;
        return -1;
      }
      g_cache.emplace(src, c);
    }
  }
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
      r = get(&f, m, "spx_ewj");
      if (r != CUDA_SUCCESS) return spx_set_error("ew jit: cuModuleGetFunction failed (%d)", (int)r);
      j->c->fn.emplace(dev, f);
    }
  }
  CUlaunchConfig cfg = {};
  cfg.gridDimX = j->blocks;
  cfg.gridDimY = j->ndev;
  cfg.gridDimZ = 1;
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

int spx_ew_jit_stats(int* compiles, int* cached) {
  std::lock_guard<std::mutex> lk(g_mu);
  *compiles = g_compiles;
  *cached = (int)g_cache.size();
  return 0;
}

}  // extern "C"
