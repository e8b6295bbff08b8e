// All-reduce over NVLink peer memory (one mesh device per process, arenas
// mapped into every peer with CUDA IPC).  For the latency-bound collectives on
// the critical path (the Megatron activation reductions: ~4 MB, 32-64 per C2
// step) a one-shot all-reduce beats a ring: every rank reads the n-1 peer
// inputs straight over NVLink and folds them IN MEMBER ORDER -- the left fold
// of the reference's `_combine` (spmd_interp.py:66-71) -- so every replica
// gets bit-identical values, identical to the reference evaluator's.
//
// One launch.  Block b of every member owns the same slice of the tensor and
// synchronises only with block b of the other members, through per-block
// flag words in every member's arena (written remotely):
//   1. arrive: store epoch into flags[slot][0][b][me] of every member, wait
//      until all members' block b arrived (their inputs are complete: the
//      kernel runs after its producers in stream order);
//   2. out[i] = src[0][i] + src[1][i] + ... for the block's slice (float4, all
//      members' loads in flight before the fold);
//   3. depart: store epoch into flags[slot][1][b][me] of every member, wait
//      until all members' block b are done reading -- nobody leaves (and may
//      overwrite its input) while a peer still reads it.
// Epochs are per (slot, block) counters in the local arena, so graph replays
// and eager runs keep counting without host involvement.
//
// Forward progress.  A block spins until the same block of every member has
// arrived, so a member must never let one peer kernel starve another of SM
// slots: with two slots in flight (main and collective streams), rank A may
// start X before Y and rank B Y before X.  Hence (1) a peer kernel never lets
// its stream's NEXT kernel launch early (no PDL trigger before the final
// barrier: PDL dependents parked at griddepcontrol.wait would fill the SMs
// while X waits on a peer), and (2) a peer kernel holds at most one block per
// SM while every variant fits two per SM (__launch_bounds__(256, 2)), so a
// second peer kernel -- or an NCCL kernel -- always finds room.
#include <cstdlib>
#include <cstring>
#include "common.cuh"

namespace {

// Flag protocol and memory ordering.  Flags are written with system-scope
// stores into the members' arenas and polled with relaxed system-scope loads.
// Where a barrier publishes data written IN THE SAME KERNEL (the two-shot
// all-reduce's reduced segments, read by the peers after phase 1) the block
// fences at system scope between its writes and its flag stores, and again
// between its successful polls and its reads of the peers' data: the
// fence-based message-passing pattern of the PTX model (bar.sync makes the
// other threads' writes/reads part of the release/acquire).  The arrive barrier of phase 0
// publishes inputs completed by EARLIER kernels (kernel boundaries) and the
// depart barrier orders only reads before a later overwrite (every load of
// the block has returned when __syncthreads completes), so those use relaxed
// flags unless SPX_PEER_ORDER=2 asks for release/acquire everywhere
// (SPX_PEER_ORDER=0: relaxed everywhere, the round-1 protocol).
SPX_DEV void st_flag(uint32_t* p, uint32_t v, bool release) {
  if (release) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SPX_DEV uint32_t ld_flag(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SPX_DEV uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Set when a barrier gave up waiting (a member never arrived within the
// timeout): the kernel abandons the wait -- its results are garbage -- and the
// host raises (spx_peer_error, polled while the host waits for the stream)
// instead of the context dying on a trap.  The word lives in mapped pinned host
// memory, so the host reads it without any CUDA call.
uint32_t* g_err_host = nullptr;
uint32_t* g_err_dev = nullptr;

// flag word of (slot, phase, block, member) inside a member's flag region
SPX_DEV uint32_t* flag_at(uint64_t region, int slot, int phase, int block, int member) {
  return reinterpret_cast<uint32_t*>(region) +
         (((int64_t)(slot * SPX_PEER_PHASES + phase) * SPX_PEER_MAX_BLOCKS + block) * 8 + member);
}

struct PeerSync {
  uint64_t timeout_ns;   // 0: wait forever
  int order;             // SPX_PEER_ORDER
  uint32_t* err;         // mapped host error word
};

// publish: this barrier makes data written by this kernel visible to the peers.
// SPX_PEER_ORDER: 0 relaxed everywhere; 1 (default) release/acquire at system
// scope on publishing barriers -- one fence.acq_rel.sys per block on each side
// (after the block's __syncthreads, before the relaxed flag stores / after the
// polls), the fence-based form of the release/acquire pattern; 2 the same on
// every barrier; 3 publishing barriers at GPU scope (fence.acq_rel.gpu:
// sufficient in practice, since a peer reads this GPU's memory through this
// GPU's L2, but outside the PTX model's cross-GPU rules -- measurement only).
SPX_DEV void block_barrier(const spx_peer_params& p, int phase, uint32_t epoch, PeerSync ps, bool publish) {
  const int t = threadIdx.x;
  const bool ra = ps.order == 2 || ((ps.order == 1 || ps.order == 3) && publish);
  const bool gpu = ps.order == 3;
  if (ra) {
    // every thread's writes are ordered before thread 0's fence by the caller's
    // __syncthreads; the fence orders them before the flag stores below
    if (t == 0) {
      if (gpu) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      else asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    __syncthreads();
  }
  if (t < p.n) {
    st_flag(flag_at(p.flags[t], p.slot, phase, blockIdx.x, p.me), epoch, false);
    const uint32_t* mine = flag_at(p.flags[p.me], p.slot, phase, blockIdx.x, t);
    if (ld_flag(mine) < epoch) {
      const uint64_t t0 = globaltimer();
      while (ld_flag(mine) < epoch) {
        if (ps.timeout_ns && globaltimer() - t0 > ps.timeout_ns) {
          *reinterpret_cast<volatile uint32_t*>(ps.err) = 1u + (uint32_t)phase;
          __threadfence_system();
          break;
        }
      }
    }
  }
  __syncthreads();
  if (ra) {
    // acquire: the polls (relaxed) observed the peers' flags; one fence orders
    // this block's subsequent reads of their data after them
    if (t == 0) {
      if (gpu) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      else asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    __syncthreads();
  }
}

SPX_DEV float4 fold4(int monoid, float4 a, float4 v) {
  if (monoid == 0) {
    a.x = f_add(a.x, v.x); a.y = f_add(a.y, v.y); a.z = f_add(a.z, v.z); a.w = f_add(a.w, v.w);
  } else {
    a.x = f_max(a.x, v.x); a.y = f_max(a.y, v.y); a.z = f_max(a.z, v.z); a.w = f_max(a.w, v.w);
  }
  return a;
}

// float4 per thread per iteration (loads in flight per member): N * U float4
// registers, kept under the 128-register cap of two blocks per SM
template <int N>
struct PeerU { static constexpr int value = N >= 8 ? 2 : 4; };

// wait for the previous grid; no early launch of the next one (see above)
#define SPX_PEER_ENTRY() asm volatile("griddepcontrol.wait;" ::: "memory")
#define SPX_PEER_EXIT() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")

// N > 0: member count known at compile time (all loads issued before folding)
template <int N>
__global__ void __launch_bounds__(256, 2) peer_allreduce(const __grid_constant__ spx_peer_params p, int64_t per_block,
                                                      int dbg, PeerSync ps) {
  SPX_PEER_ENTRY();
  constexpr int U = PeerU<N>::value;
  const int n = N > 0 ? N : p.n;
  uint32_t* counter = reinterpret_cast<uint32_t*>(p.counter) + (int64_t)p.slot * SPX_PEER_MAX_BLOCKS + blockIdx.x;
  const uint32_t epoch = *counter + 1u;
  if (!(dbg & 1)) block_barrier(p, 0, epoch, ps, false);
  if (dbg & 4) per_block = 0;

  const int64_t n4 = p.count >> 2;
  const int64_t b0 = (int64_t)blockIdx.x * per_block, b1 = min(n4, b0 + per_block);
  float4* dst = reinterpret_cast<float4*>(p.dst);
  for (int64_t i0 = b0 + threadIdx.x; i0 < b1; i0 += 256 * U) {
    float4 v[N > 0 ? N : 1][U];
    if (N > 0) {
#pragma unroll
      for (int m = 0; m < (N > 0 ? N : 1); ++m)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i = i0 + u * 256;
          if (i < b1) v[m][u] = reinterpret_cast<const float4*>(p.src[m])[i];
        }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * 256;
        if (i >= b1) continue;
        float4 acc = v[0][u];
#pragma unroll
        for (int m = 1; m < (N > 0 ? N : 1); ++m) acc = fold4(p.monoid, acc, v[m][u]);
        dst[i] = acc;
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * 256;
        if (i >= b1) continue;
        float4 acc = reinterpret_cast<const float4*>(p.src[0])[i];
        for (int m = 1; m < n; ++m) acc = fold4(p.monoid, acc, reinterpret_cast<const float4*>(p.src[m])[i]);
        dst[i] = acc;
      }
    }
  }
  // tail (count % 4) in the last block
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < (p.count & 3)) {
    const int64_t i = n4 * 4 + threadIdx.x;
    float acc = reinterpret_cast<const float*>(p.src[0])[i];
    for (int m = 1; m < n; ++m) {
      const float x = reinterpret_cast<const float*>(p.src[m])[i];
      acc = p.monoid == 0 ? f_add(acc, x) : f_max(acc, x);
    }
    reinterpret_cast<float*>(p.dst)[i] = acc;
  }
  __syncthreads();
  if (!(dbg & 2)) block_barrier(p, 1, epoch, ps, false);
  if (threadIdx.x == 0) *counter = epoch;
  SPX_PEER_EXIT();
}

// Two-shot (n >= 4): block b owns chunk b of every member's segment.
//   1. arrive (phase 0), then reduce chunk b of MY segment over all members'
//      inputs in member order into my output;
//   2. barrier (phase 1): every member's chunk b of its own segment is final;
//   3. copy chunk b of every other member's segment from its output;
//   4. depart (phase 2).
// NVLink traffic per rank 2(n-1)/n of the tensor instead of (n-1); the fold
// (and so every replica's bits) is the same as the one-shot kernel's.
template <int N>
__global__ void __launch_bounds__(256, 2) peer_allreduce_2shot(const __grid_constant__ spx_peer_params p,
                                                            int64_t seg4, int64_t per_block, PeerSync ps) {
  SPX_PEER_ENTRY();
  constexpr int U = PeerU<N>::value;
  uint32_t* counter = reinterpret_cast<uint32_t*>(p.counter) + (int64_t)p.slot * SPX_PEER_MAX_BLOCKS + blockIdx.x;
  const uint32_t epoch = *counter + 1u;
  block_barrier(p, 0, epoch, ps, false);
  // phase A: my segment's chunk b
  {
    const int64_t s0 = (int64_t)p.me * seg4;
    const int64_t b0 = s0 + (int64_t)blockIdx.x * per_block;
    const int64_t b1 = min(s0 + seg4, b0 + per_block);
    float4* dst = reinterpret_cast<float4*>(p.dst);
    for (int64_t i0 = b0 + threadIdx.x; i0 < b1; i0 += 256 * U) {
      float4 v[N][U];
#pragma unroll
      for (int m = 0; m < N; ++m)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i = i0 + u * 256;
          if (i < b1) v[m][u] = reinterpret_cast<const float4*>(p.src[m])[i];
        }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * 256;
        if (i >= b1) continue;
        float4 acc = v[0][u];
#pragma unroll
        for (int m = 1; m < N; ++m) acc = fold4(p.monoid, acc, v[m][u]);
        dst[i] = acc;
      }
    }
  }
  __syncthreads();
  block_barrier(p, 1, epoch, ps, true);     // my reduced segment is read by the peers next
  // phase B: the other members' chunk b, from their outputs (same arena offset)
  {
    float4* dst = reinterpret_cast<float4*>(p.dst);
    const int64_t dst_off = (int64_t)(p.dst - p.src[p.me]);    // bytes from my input to my output
#pragma unroll 1
    for (int k = 1; k < N; ++k) {
      const int m = (p.me + k) % N;
      const float4* rem = reinterpret_cast<const float4*>(p.src[m] + dst_off);
      const int64_t s0 = (int64_t)m * seg4;
      const int64_t b0 = s0 + (int64_t)blockIdx.x * per_block;
      const int64_t b1 = min(s0 + seg4, b0 + per_block);
      for (int64_t i0 = b0 + threadIdx.x; i0 < b1; i0 += 256 * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + u * 256 < b1) v[u] = rem[i0 + u * 256];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + u * 256 < b1) dst[i0 + u * 256] = v[u];
      }
    }
  }
  __syncthreads();
  block_barrier(p, 2, epoch, ps, false);
  if (threadIdx.x == 0) *counter = epoch;
  SPX_PEER_EXIT();
}

// All-gather: dst[m * count + i] = member m's src[i] (chunks in member order,
// the reference's all_gather layout for a dim-0 gather in group order).  The
// same arrive / depart barriers: inputs complete before anyone reads, nobody
// leaves while a peer still reads its input.
template <int N>
__global__ void __launch_bounds__(256, 2) peer_allgather(const __grid_constant__ spx_peer_params p, int64_t per_block,
                                                      PeerSync ps) {
  SPX_PEER_ENTRY();
  constexpr int U = PeerU<N>::value;
  uint32_t* counter = reinterpret_cast<uint32_t*>(p.counter) + (int64_t)p.slot * SPX_PEER_MAX_BLOCKS + blockIdx.x;
  const uint32_t epoch = *counter + 1u;
  block_barrier(p, 0, epoch, ps, false);
  const int64_t n4 = p.count >> 2;
  const int64_t b0 = (int64_t)blockIdx.x * per_block, b1 = min(n4, b0 + per_block);
  float4* dst = reinterpret_cast<float4*>(p.dst);
  for (int64_t i0 = b0 + threadIdx.x; i0 < b1; i0 += 256 * U) {
    float4 v[N][U];
#pragma unroll
    for (int m = 0; m < N; ++m)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * 256;
        if (i < b1) v[m][u] = reinterpret_cast<const float4*>(p.src[m])[i];
      }
#pragma unroll
    for (int m = 0; m < N; ++m)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * 256;
        if (i < b1) dst[m * n4 + i] = v[m][u];
      }
  }
  __syncthreads();
  block_barrier(p, 1, epoch, ps, false);
  if (threadIdx.x == 0) *counter = epoch;
  SPX_PEER_EXIT();
}

// One-block barrier (kind 3): every member arrives and waits for the others --
// the handshakes around the copy-engine reduce-scatter (inputs complete /
// inputs released).  Holds one SM while it waits.
__global__ void __launch_bounds__(32) peer_barrier_kernel(const __grid_constant__ spx_peer_params p, PeerSync ps) {
  SPX_PEER_ENTRY();
  uint32_t* counter = reinterpret_cast<uint32_t*>(p.counter) + (int64_t)p.slot * SPX_PEER_MAX_BLOCKS;
  const uint32_t epoch = *counter + 1u;
  block_barrier(p, 0, epoch, ps, false);
  if (threadIdx.x == 0) *counter = epoch;
  SPX_PEER_EXIT();
}

}  // namespace

static int peer_err_init() {
  if (g_err_host) return 0;
  void* h = nullptr;
  SPX_CUDA(cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 0, 64);
  void* d = nullptr;
  SPX_CUDA(cudaHostGetDevicePointer(&d, h, 0));
  g_err_host = static_cast<uint32_t*>(h);
  g_err_dev = static_cast<uint32_t*>(d);
  return 0;
}

// 0: no peer barrier has timed out; else 1 + the phase that gave up
extern "C" int spx_peer_error(int* out) {
  *out = g_err_host ? (int)*reinterpret_cast<volatile uint32_t*>(g_err_host) : 0;
  return 0;
}

extern "C" int spx_peer_error_clear(void) {
  if (g_err_host) *reinterpret_cast<volatile uint32_t*>(g_err_host) = 0;
  return 0;
}

int spx_launch_peer(const spx_peer_params& p, cudaStream_t s, int* nlaunch) {
  if (p.n < 1 || p.n > 8) return spx_set_error("peer collective: group size %d", p.n);
  if (p.kind == 3) {
    static PeerSync bs = {~0ull, -1, nullptr};
    if (bs.order < 0) {
      if (peer_err_init()) return -1;
      bs.err = g_err_dev;
      const char* t = getenv("SPX_PEER_TIMEOUT_S");
      const double sec = t ? atof(t) : 300.0;
      bs.timeout_ns = sec > 0 ? (uint64_t)(sec * 1e9) : 0;
      bs.order = 0;     // the inputs were completed by earlier kernels; the copies are stream-ordered
    }
    spx_launch(peer_barrier_kernel, dim3(1), 32, 0, s, p, bs);
    SPX_CHECK_LAUNCH();
    if (nlaunch) ++*nlaunch;
    return 0;
  }
  if ((p.dst & 15) || p.kind < 0 || p.kind > 2 || (p.kind == 1 && (p.count & 3)))
    return spx_set_error("peer collective: unsupported record");
  for (int m = 0; m < p.n; ++m)
    if (p.src[m] & 15) return spx_set_error("peer collective: unaligned source");
  // blocks: ~2 float4 per thread, at most one per SM (forward progress, see
  // the top of the file) and SPX_PEER_MAX_BLOCKS (flag space); identical on
  // every member
  const int64_t n4 = p.count >> 2;
  int64_t blocks = (n4 + 256 * 2 - 1) / (256 * 2);
  static int per_sm = -1;
  if (per_sm < 0) { const char* e = getenv("SPX_PEER_BLOCKS_PER_SM"); per_sm = e ? atoi(e) : 1; }
  int64_t cap = (int64_t)spx_num_sms() * per_sm < SPX_PEER_MAX_BLOCKS ? (int64_t)spx_num_sms() * per_sm : SPX_PEER_MAX_BLOCKS;
  if (p.max_blocks > 0 && p.max_blocks < cap) cap = p.max_blocks;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const int64_t per_block = (n4 + blocks - 1) / blocks;
  static PeerSync ps = {~0ull, -1, nullptr};
  if (ps.order < 0) {
    if (peer_err_init()) return -1;
    ps.err = g_err_dev;
    const char* e = getenv("SPX_PEER_ORDER");
    ps.order = e ? atoi(e) : 1;
    const char* t = getenv("SPX_PEER_TIMEOUT_S");
    const double sec = t ? atof(t) : 300.0;
    ps.timeout_ns = sec > 0 ? (uint64_t)(sec * 1e9) : 0;
  }
  static int dbg = -1, two = -1;
  if (dbg < 0) { const char* e = getenv("SPX_PEER_DBG"); dbg = e ? atoi(e) : 0; }
  if (two < 0) { const char* e = getenv("SPX_PEER_TWOSHOT"); two = e ? atoi(e) : 1; }
  // two-shot for 4 and 8 members from 2 MB (4 ranks, 4 MB: 18.7 us vs 25.0 us
  // one-shot; 1 MB: 14.4 vs 11.2), when every segment is whole float4s
  if (p.kind == 1) {
    switch (p.n) {
      case 2: spx_launch(peer_allgather<2>, dim3((unsigned)blocks), 256, 0, s, p, per_block, ps); break;
      case 3: spx_launch(peer_allgather<3>, dim3((unsigned)blocks), 256, 0, s, p, per_block, ps); break;
      case 4: spx_launch(peer_allgather<4>, dim3((unsigned)blocks), 256, 0, s, p, per_block, ps); break;
      case 8: spx_launch(peer_allgather<8>, dim3((unsigned)blocks), 256, 0, s, p, per_block, ps); break;
      default: return spx_set_error("peer all-gather: group size %d", p.n);
    }
    SPX_CHECK_LAUNCH();
    if (nlaunch) ++*nlaunch;
    return 0;
  }
  // kind 2, reduce-scatter: the sources point at this member's chunk of every
  // member's input, and only that chunk is folded (one-shot kernel)
  // two-shot from 2 MB with 8 members; with 4 from 8 MB: its publishing barrier's
  // system-scope fences (release/acquire, SPX_PEER_ORDER=1) cost ~9 us, so below
  // that the one-shot kernel is faster (profiles/r02_peer_order_variants.txt:
  // 4 MB 26.1 vs 28.4 us, 16 MB 89.3 vs 57.9 us)
  const int64_t two_min = (p.n == 4 && ps.order != 0 && ps.order != 3) ? (int64_t)524288 : (int64_t)131072;
  if (two && p.kind == 0 && p.max_blocks == 0 && (p.n == 4 || p.n == 8) && (p.count & 3) == 0 && (n4 % p.n) == 0 && n4 >= two_min && !dbg) {
    const int64_t seg4 = n4 / p.n;
    int64_t b2 = (seg4 + 256 * 2 - 1) / (256 * 2);     // ~2 float4 per thread per phase
    if (b2 > cap) b2 = cap;
    if (b2 < 1) b2 = 1;
    const int64_t pb = (seg4 + b2 - 1) / b2;
    if (p.n == 4) spx_launch(peer_allreduce_2shot<4>, dim3((unsigned)b2), 256, 0, s, p, seg4, pb, ps);
    else spx_launch(peer_allreduce_2shot<8>, dim3((unsigned)b2), 256, 0, s, p, seg4, pb, ps);
    SPX_CHECK_LAUNCH();
    if (nlaunch) ++*nlaunch;
    return 0;
  }
  switch (p.n) {
    case 2: spx_launch(peer_allreduce<2>, dim3((unsigned)blocks), 256, 0, s, p, per_block, dbg, ps); break;
    case 4: spx_launch(peer_allreduce<4>, dim3((unsigned)blocks), 256, 0, s, p, per_block, dbg, ps); break;
    case 8: spx_launch(peer_allreduce<8>, dim3((unsigned)blocks), 256, 0, s, p, per_block, dbg, ps); break;
    default: spx_launch(peer_allreduce<0>, dim3((unsigned)blocks), 256, 0, s, p, per_block, dbg, ps);
  }
  SPX_CHECK_LAUNCH();
  if (nlaunch) ++*nlaunch;
  return 0;
}
