// Shared device helpers for the spindle_b200 kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "spindle_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "spindle_b200 kernels target sm_100a (Blackwell) only"
#endif

#include <utility>
#define SPX_DEV __device__ __forceinline__

// Arena addressing: device d's copy of an element offset.
SPX_DEV float* dev_ptr(uint64_t base, int64_t dev_stride, int d, int64_t off) {
  return reinterpret_cast<float*>(base + (uint64_t)((int64_t)d * dev_stride) + (uint64_t)(off * 4));
}

// IEEE fp32 ops with explicit rounding so ptxas never contracts a*b+c into an
// FMA: numpy evaluates each elementwise op separately, and bit-exact parity
// with it (interp.py:45-48) needs the same per-op rounding.
SPX_DEV float f_add(float a, float b) { return __fadd_rn(a, b); }
SPX_DEV float f_mul(float a, float b) { return __fmul_rn(a, b); }
// np.maximum: NaN in either operand propagates.
SPX_DEV float f_max(float a, float b) { return (a != a || a > b) ? a : b; }

SPX_DEV float apply_op(int op, float a, float b, float imm) {
  switch (op) {
    case SPX_OP_MOV: return a;
    case SPX_OP_ADD: return f_add(a, b);
    case SPX_OP_MUL: return f_mul(a, b);
    case SPX_OP_NEG: return -a;
    case SPX_OP_EXP: return expf(a);
    case SPX_OP_MAX: return f_max(a, b);
    case SPX_OP_IMM: return imm;
    case SPX_OP_ADDI: return f_add(a, imm);
    case SPX_OP_MULI: return f_mul(a, imm);
    case SPX_OP_IADD: return f_add(imm, a);
    case SPX_OP_IMUL: return f_mul(imm, a);
  }
  return 0.f;
}

// Host-side error plumbing (defined in runtime.cu).
#ifndef __CUDACC_RTC__
int spx_set_error(const char* fmt, ...);
#define SPX_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess)                                                    \
      return spx_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,        \
                           cudaGetErrorString(_e));                           \
  } while (0)
#define SPX_CHECK_LAUNCH() SPX_CUDA(cudaGetLastError())
#endif

// Launch entry points (host) implemented per kernel family.
int spx_launch_ew(const spx_ew_params& p, cudaStream_t s, int* nlaunch);
int spx_ew_static_match(const spx_ew_params& p);     // catalog index or -1 (ew_static.cu)
int spx_launch_ew_static(int id, const spx_ew_params& p, cudaStream_t s, int* nlaunch);
struct SpxEwJit;                                      // run-time specialised kernel (ew_jit.cu)
bool spx_ew_jit_enabled();
int spx_ew_jit_prepare(const spx_ew_params& p, SpxEwJit** out);
int spx_ew_jit_launch(const SpxEwJit* j, cudaStream_t s, int* nlaunch);
void spx_ew_jit_free(SpxEwJit* j);
int spx_ew_jit_split_prepare(const spx_ew_params& p, const spx_split_params& sp, int which, int skip, SpxEwJit** out);
int spx_launch_reduce(const spx_reduce_params& p, cudaStream_t s, int* nlaunch);
int spx_launch_gather(const spx_gather_params& p, cudaStream_t s, int* nlaunch);
int spx_launch_creduce(const spx_creduce_params& p, cudaStream_t s, int* nlaunch);
int spx_launch_gemm_simt(const spx_gemm_params& p, cudaStream_t s, int* nlaunch);
int spx_launch_peer(const spx_peer_params& p, cudaStream_t s, int* nlaunch);
// int32 arithmetic records (int32.cu)
int spx_launch_ew_i32(const spx_ew_params& p, cudaStream_t s, int* nlaunch);
int spx_launch_reduce_i32(const spx_reduce_params& p, cudaStream_t s, int* nlaunch);
int spx_launch_creduce_i32(const spx_creduce_params& p, cudaStream_t s, int* nlaunch);
int spx_launch_gemm_i32(const spx_gemm_params& p, cudaStream_t s, int* nlaunch);

struct SpxGemmTC;  // prepared tcgen05 GEMM (tensor maps), see gemm_tc.cu
int spx_gemm_tc_prepare(const spx_gemm_params& p, SpxGemmTC** out);
int spx_gemm_tc_launch(const SpxGemmTC* g, cudaStream_t s, int* nlaunch);
void spx_gemm_tc_free(SpxGemmTC* g);
bool spx_gemm_tc_supported(const spx_gemm_params& p);

struct SpxGemmH3;  // prepared block-scaled 3xFP16 GEMM, see gemm_h3.cu
bool spx_gemm_h3_supported(const spx_gemm_params& p);
int spx_gemm_h3_prepare(const spx_gemm_params& p, SpxGemmH3** out);
int64_t spx_gemm_h3_ws_bytes(const SpxGemmH3* g);
int spx_gemm_h3_bind(SpxGemmH3* g, uint64_t ws);
int spx_gemm_h3_launch(const SpxGemmH3* g, cudaStream_t s, int* nlaunch);
void spx_gemm_h3_free(SpxGemmH3* g);
int spx_launch_split(const spx_split_params& p, cudaStream_t s, int* nlaunch);
int spx_launch_split_batch(const spx_split_params* const* p, int n, cudaStream_t s, int* nlaunch);
int spx_split_batch_max(void);
int spx_ew_split_match(const spx_ew_params& p, const spx_split_params& sp);
int spx_launch_ew_static_split(int id, const spx_ew_params& p, const spx_split_params& sp, int which,
                               cudaStream_t s, int* nlaunch);

int spx_num_sms();
int spx_h3_range_split(uint32_t* out, int reset);   // gemm_h3.cu
int spx_h3_range_ew(uint32_t* out, int reset);      // ew_static.cu

// Programmatic dependent launch: every kernel starts with SPX_PDL_ENTRY --
// it lets the NEXT kernel in the stream be scheduled once all of this grid's
// CTAs are running (its launch latency and prologue then overlap our tail),
// and waits for the PREVIOUS grid's completion (and memory) before touching
// global memory.  Kernels launched through spx_launch carry the attribute;
// without it (SPX_PDL=0, or a non-PDL predecessor such as an NCCL kernel) the
// wait returns immediately and ordering is plain stream order.
#define SPX_PDL_ENTRY() asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory")
bool spx_pdl_enabled();

template <typename... KArgs, typename... Args>
inline void spx_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = spx_pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
