// All-reduce over NVLink peer memory (one mesh device per process, arenas
// mapped into every peer with CUDA IPC).  For the latency-bound collectives on
// the critical path (the Megatron activation reductions: ~4 MB, 64 per C2
// step) a one-shot all-reduce beats a ring: every rank reads the n-1 peer
// inputs straight over NVLink and folds them IN MEMBER ORDER -- the left fold
// of the reference's `_combine` (spmd_interp.py:66-71) -- so every replica
// gets bit-identical values, identical to the reference evaluator's.
//
// One record = three launches on the stream:
//   1. peer_barrier  (1 warp): epoch = ++counter[slot]; store epoch into every
//      member's flag word for (slot, phase 0, me) with st.release.sys, spin
//      (bounded, traps on timeout) until all members' words reach epoch --
//      every member's input is complete;
//   2. peer_sum: out[i] = src[0][i] + src[1][i] + ... (float4, grid-stride);
//   3. peer_barrier phase 1: nobody proceeds (and may overwrite its input)
//      until every member has finished reading.
#include "common.cuh"

namespace {

SPX_DEV void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SPX_DEV uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// flag word address of (slot, phase, member) inside a rank's flag region
SPX_DEV uint32_t* flag_at(uint64_t region, int slot, int phase, int member) {
  return reinterpret_cast<uint32_t*>(region) + ((slot * 2 + phase) * 8 + member);
}

__global__ void peer_barrier(const __grid_constant__ spx_peer_params p, int phase) {
  const int lane = threadIdx.x;
  uint32_t* counter = reinterpret_cast<uint32_t*>(p.counter) + p.slot;
  uint32_t epoch = 0;
  if (lane == 0) {
    epoch = *counter + (phase == 0 ? 1u : 0u);
    if (phase == 0) *counter = epoch;
  }
  epoch = __shfl_sync(0xffffffffu, epoch, 0);
  __threadfence_system();
  if (lane < p.n) st_release_sys(flag_at(p.flags[lane], p.slot, phase, p.me), epoch);
  if (lane < p.n) {
    const uint32_t* mine = flag_at(p.flags[p.me], p.slot, phase, lane);
    long long t0 = clock64();
    while (ld_acquire_sys(mine) < epoch) {
      __nanosleep(64);
      if (clock64() - t0 > 20000000000LL) __trap();     // ~10 s: a peer never arrived
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256) peer_sum(const __grid_constant__ spx_peer_params p) {
  const int64_t n4 = p.count >> 2;
  float4* dst = reinterpret_cast<float4*>(p.dst);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(p.src[0])[i];
    for (int m = 1; m < p.n; ++m) {
      const float4 v = reinterpret_cast<const float4*>(p.src[m])[i];
      if (p.monoid == 0) {
        acc.x = f_add(acc.x, v.x); acc.y = f_add(acc.y, v.y); acc.z = f_add(acc.z, v.z); acc.w = f_add(acc.w, v.w);
      } else {
        acc.x = f_max(acc.x, v.x); acc.y = f_max(acc.y, v.y); acc.z = f_max(acc.z, v.z); acc.w = f_max(acc.w, v.w);
      }
    }
    dst[i] = acc;
  }
  // tail (count % 4)
  if (blockIdx.x == 0 && threadIdx.x < (p.count & 3)) {
    const int64_t i = n4 * 4 + threadIdx.x;
    float acc = reinterpret_cast<const float*>(p.src[0])[i];
    for (int m = 1; m < p.n; ++m) {
      const float v = reinterpret_cast<const float*>(p.src[m])[i];
      acc = p.monoid == 0 ? f_add(acc, v) : f_max(acc, v);
    }
    reinterpret_cast<float*>(p.dst)[i] = acc;
  }
}

}  // namespace

int spx_launch_peer(const spx_peer_params& p, cudaStream_t s, int* nlaunch) {
  if (p.n < 1 || p.n > 8) return spx_set_error("peer collective: group size %d", p.n);
  if ((p.dst & 15) || p.kind != 0) return spx_set_error("peer collective: unsupported record");
  for (int m = 0; m < p.n; ++m)
    if (p.src[m] & 15) return spx_set_error("peer collective: unaligned source");
  peer_barrier<<<1, 32, 0, s>>>(p, 0);
  SPX_CHECK_LAUNCH();
  int64_t b = (p.count / 4 + 255) / 256;
  const int64_t cap = (int64_t)spx_num_sms() * 4;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  peer_sum<<<(unsigned)b, 256, 0, s>>>(p);
  SPX_CHECK_LAUNCH();
  peer_barrier<<<1, 32, 0, s>>>(p, 1);
  SPX_CHECK_LAUNCH();
  if (nlaunch) *nlaunch += 3;
  return 0;
}
