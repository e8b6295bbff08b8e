// Host runtime of the C-ABI (include/spindle_b200.h): device/arena/stream
// management, plan records -> kernel launches, CUDA-graph capture of a whole
// partitioned step, NCCL (dlopen'd, the same libnccl torch loads) for
// collectives that cross processes.
#include <dlfcn.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <nvtx3/nvToolsExt.h>
#include "common.cuh"

static thread_local char g_err[1024] = "";

// NVTX range per issued record (SPX_NVTX=1): "gemm 8192x8192x2048", "ew",
// "peer all_reduce" ... -- for ncu --nvtx-include / Nsight timelines; header-only
// NVTX3, a no-op unless a tool is attached
static bool nvtx_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SPX_NVTX");
    on = e ? atoi(e) != 0 : 0;
  }
  return on != 0;
}

int spx_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return -1;
}

// spins for `ns` nanoseconds of the global timer (profile mode: see spx_plan_profile)
__global__ void hold_stream_kernel(long long ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(10000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((long long)(t - t0) < ns);
}

static int g_num_sms = 148;
int spx_num_sms() { return g_num_sms; }
// GEMMs the plan leaves to the backend (path 0) take the block-scaled 3xFP16
// kernel where it applies; SPX_GEMM_H3=0 keeps them on 3xTF32.
static bool h3_default() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SPX_GEMM_H3");
    on = e ? atoi(e) != 0 : 1;
  }
  return on != 0;
}

bool spx_pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SPX_PDL");
    on = e ? atoi(e) != 0 : 1;
  }
  return on != 0;
}

// ---------------------------------------------------------------------------
// NCCL via dlopen (no link-time dependency; reuse the process's libnccl)
// ---------------------------------------------------------------------------
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
typedef int (*fn_get_uid)(nccl_uid_t*);
typedef int (*fn_init_rank)(nccl_comm_t*, int, nccl_uid_t, int);
typedef int (*fn_destroy)(nccl_comm_t);
typedef int (*fn_allreduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_allgather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_reducescatter)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_sendrecv)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_group)(void);
typedef const char* (*fn_errstr)(int);
typedef int (*fn_count)(nccl_comm_t, int*);
typedef int (*fn_async)(nccl_comm_t, int*);
typedef int (*fn_abort)(nccl_comm_t);

static struct {
  void* h = nullptr;
  fn_get_uid get_uid;
  fn_init_rank init_rank;
  fn_destroy destroy;
  fn_allreduce allreduce;
  fn_allgather allgather;
  fn_reducescatter reducescatter;
  fn_sendrecv send, recv;
  fn_group gstart, gend;
  fn_errstr errstr;
  fn_count count;
  fn_async async_error;
  fn_abort abort;
} N;
static std::vector<nccl_comm_t> g_comms;

static int nccl_load() {
  if (N.h) return 0;
  const char* env = getenv("SPX_NCCL_LIB");
  const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char* c : cands) {
    if (!c) continue;
    N.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (N.h) break;
  }
  if (!N.h) return spx_set_error("cannot dlopen libnccl (set SPX_NCCL_LIB)");
#define LOADSYM(field, name)                                            \
  N.field = reinterpret_cast<decltype(N.field)>(dlsym(N.h, name));      \
  if (!N.field) return spx_set_error("libnccl lacks %s", name);
  LOADSYM(get_uid, "ncclGetUniqueId");
  LOADSYM(init_rank, "ncclCommInitRank");
  LOADSYM(destroy, "ncclCommDestroy");
  LOADSYM(allreduce, "ncclAllReduce");
  LOADSYM(allgather, "ncclAllGather");
  LOADSYM(reducescatter, "ncclReduceScatter");
  LOADSYM(send, "ncclSend");
  LOADSYM(recv, "ncclRecv");
  LOADSYM(gstart, "ncclGroupStart");
  LOADSYM(gend, "ncclGroupEnd");
  LOADSYM(errstr, "ncclGetErrorString");
  LOADSYM(count, "ncclCommCount");
  LOADSYM(async_error, "ncclCommGetAsyncError");
  LOADSYM(abort, "ncclCommAbort");
#undef LOADSYM
  return 0;
}

#define SPX_NCCL(call)                                                              \
  do {                                                                              \
    int _r = (call);                                                                \
    if (_r != 0) return spx_set_error("%s: nccl error %d (%s)", #call, _r, N.errstr(_r)); \
  } while (0)

static const int NCCL_FLOAT = 7, NCCL_SUM = 0, NCCL_MAX = 2;

static int run_nccl(const spx_nccl_params& p, cudaStream_t s) {
  if (p.comm < 0 || p.comm >= (int)g_comms.size() || !g_comms[p.comm]) return spx_set_error("bad comm %d", p.comm);
  nccl_comm_t c = g_comms[p.comm];
  const int op = p.monoid == 0 ? NCCL_SUM : NCCL_MAX;
  const void* sb = reinterpret_cast<const void*>(p.send);
  void* rb = reinterpret_cast<void*>(p.recv);
  switch (p.kind) {
    case SPX_NCCL_ALLREDUCE: SPX_NCCL(N.allreduce(sb, rb, (size_t)p.count, NCCL_FLOAT, op, c, s)); break;
    case SPX_NCCL_ALLGATHER: SPX_NCCL(N.allgather(sb, rb, (size_t)p.count, NCCL_FLOAT, c, s)); break;
    case SPX_NCCL_REDUCESCATTER: SPX_NCCL(N.reducescatter(sb, rb, (size_t)p.count, NCCL_FLOAT, op, c, s)); break;
    case SPX_NCCL_ALLTOALL: {
      int n = 0;
      SPX_NCCL(N.count(c, &n));
      SPX_NCCL(N.gstart());
      for (int r = 0; r < n; ++r) {
        SPX_NCCL(N.send(static_cast<const float*>(sb) + (size_t)r * p.count, (size_t)p.count, NCCL_FLOAT, r, c, s));
        SPX_NCCL(N.recv(static_cast<float*>(rb) + (size_t)r * p.count, (size_t)p.count, NCCL_FLOAT, r, c, s));
      }
      SPX_NCCL(N.gend());
      break;
    }
    default: return spx_set_error("bad nccl kind %d", p.kind);
  }
  return 0;
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
struct Record {
  int kind;
  int path;  // GEMM: 1 tcgen05, 2 simt
  std::vector<uint8_t> params;
  SpxGemmTC* tc = nullptr;
  SpxGemmH3* h3 = nullptr;      // path 3: block-scaled 3xFP16 (gemm_h3.cu)
  SpxEwJit* jit = nullptr;      // EW path -3: run-time specialised kernel (ew_jit.cu)
  SpxEwJit* jit_split = nullptr;  // EW path -3 with the next record's split fused in
  int fused_split = -1;         // EW: the next record (SPX_K_SPLIT of output `split_out`) runs inside this launch
  int split_out = -1;
  std::vector<uint8_t> split_params;
  bool fused = false;           // SPLIT done by the preceding EW record, or by an earlier SPLIT record's batch
  std::vector<int> batch;       // SPLIT: later SPLIT records launched together with this one (path 2)
  std::vector<spx_split_params> batch_params;   // this record's and theirs, in record order
  int tag = 0;                  // spx_tag_bits: logical collective executed / internal work
  double flops = 0;             // simulator-convention FLOPs of one launch (all virtual devices)
  int stream = 0;               // 0 main, 1..SPX_SIDE_STREAMS side streams
  std::vector<int> waits;       // records on other streams to wait for
  bool signal = false;          // a later record on another stream waits for this one
  cudaEvent_t done = nullptr;
  cudaGraphNode_t node = nullptr;   // SPX_K_COPY: its memcpy node in the captured graph
};

constexpr int SPX_SIDE_STREAMS = 5;   // 1 off-critical compute, 2 collectives, 3 parameter updates, 4/5 H2D/D2H copies

struct Plan {
  std::vector<Record> recs;
  bool finalized = false;
  bool two_streams = false;              // any record off the main stream
  bool used[SPX_SIDE_STREAMS + 1] = {};
  cudaStream_t side[SPX_SIDE_STREAMS + 1] = {};
  cudaEvent_t fork = nullptr, join[SPX_SIDE_STREAMS + 1] = {};
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int launches = 0;
  void* h3ws[SPX_SIDE_STREAMS + 1] = {};   // fp16-pieces workspace per stream (GEMMs of a stream run in order)
  spx_exec_stats stats = {};               // issued so far
  spx_exec_stats graph_tally = {};         // issued into the captured graph (added per replay)
};

// work of the records issued since `tally` was reset
static void tally_record(const Record& r, spx_exec_stats* t) {
  if (r.fused) return;
  const int c = r.tag & SPX_TAG_COLL_MASK;
  if (c >= 1 && c <= 4) t->coll[c - 1] += 1;
  if (!(r.tag & SPX_TAG_INTERNAL)) t->flops += r.flops;
}

static bool arith_op(int op) {
  return op == SPX_OP_ADD || op == SPX_OP_MUL || op == SPX_OP_NEG || op == SPX_OP_EXP || op == SPX_OP_MAX ||
         op == SPX_OP_ADDI || op == SPX_OP_MULI || op == SPX_OP_IADD || op == SPX_OP_IMUL;
}

static double ew_flops(const spx_ew_params& p) {
  int n = 0;
  for (int i = 0; i < p.n_prog; ++i) n += arith_op(p.prog[i].op);
  return (double)n * (double)p.numel * (double)p.ndev;
}

// simulator convention (sim.py:86-100): matmul 2mkn, add/mul/neg/exp one per
// result element, reduce one per input element
static double record_flops(const Record& r) {
  switch (r.kind) {
    case SPX_K_GEMM: {
      const spx_gemm_params& g = *reinterpret_cast<const spx_gemm_params*>(r.params.data());
      // + the fused elementwise consumer's operations per output element
      const int epi = g.epi == SPX_EPI_ADD ? 1 : g.epi == SPX_EPI_SQUARE ? 1 : g.epi == SPX_EPI_MULSCALE ? 2
                    : g.epi == SPX_EPI_MOMENTUM ? 5 : 0;
      return (2.0 * g.K + epi) * g.M * (double)g.N * g.ndev;
    }
    case SPX_K_EW: return ew_flops(*reinterpret_cast<const spx_ew_params*>(r.params.data()));
    case SPX_K_REDUCE: {
      const spx_reduce_params& q = *reinterpret_cast<const spx_reduce_params*>(r.params.data());
      return ew_flops(q.x) + (double)q.x.numel * q.x.ndev;
    }
  }
  return 0.0;
}

static int run_record_impl(Record& r, cudaStream_t s, int* nl);

static const char* kind_name(int k) {
  switch (k) {
    case SPX_K_EW: return "ew";
    case SPX_K_REDUCE: return "reduce";
    case SPX_K_GEMM: return "gemm";
    case SPX_K_GATHER: return "gather";
    case SPX_K_CREDUCE: return "collective";
    case SPX_K_NCCL: return "nccl";
    case SPX_K_PEER: return "peer";
    case SPX_K_SPLIT: return "split";
    case SPX_K_COPY: return "copy";
  }
  return "record";
}

static int run_record(Record& r, cudaStream_t s, int* nl) {
  if (!nvtx_on() || r.fused) return run_record_impl(r, s, nl);
  char name[96];
  if (r.kind == SPX_K_GEMM) {
    const spx_gemm_params& g = *reinterpret_cast<const spx_gemm_params*>(r.params.data());
    snprintf(name, sizeof(name), "gemm p%d %dx%dx%d", r.path, g.M, g.N, g.K);
  } else {
    snprintf(name, sizeof(name), "%s", kind_name(r.kind));
  }
  nvtxRangePushA(name);
  const int rc = run_record_impl(r, s, nl);
  nvtxRangePop();
  return rc;
}

static int run_record_impl(Record& r, cudaStream_t s, int* nl) {
  if (r.fused) return 0;
  switch (r.kind) {
    case SPX_K_EW:
      if (reinterpret_cast<const spx_ew_params*>(r.params.data())->dtype == SPX_DT_I32)
        return spx_launch_ew_i32(*reinterpret_cast<const spx_ew_params*>(r.params.data()), s, nl);
      if (r.fused_split >= 0 && r.jit_split) return spx_ew_jit_launch(r.jit_split, s, nl);
      if (r.fused_split >= 0)
        return spx_launch_ew_static_split(r.path - 1, *reinterpret_cast<const spx_ew_params*>(r.params.data()),
                                          *reinterpret_cast<const spx_split_params*>(r.split_params.data()),
                                          r.split_out, s, nl);
      if (r.path > 0) return spx_launch_ew_static(r.path - 1, *reinterpret_cast<const spx_ew_params*>(r.params.data()), s, nl);
      if (r.jit) return spx_ew_jit_launch(r.jit, s, nl);
      return spx_launch_ew(*reinterpret_cast<const spx_ew_params*>(r.params.data()), s, nl);
    case SPX_K_REDUCE: {
      const spx_reduce_params& q = *reinterpret_cast<const spx_reduce_params*>(r.params.data());
      return q.x.dtype == SPX_DT_I32 ? spx_launch_reduce_i32(q, s, nl) : spx_launch_reduce(q, s, nl);
    }
    case SPX_K_GATHER: return spx_launch_gather(*reinterpret_cast<const spx_gather_params*>(r.params.data()), s, nl);
    case SPX_K_CREDUCE: {
      const spx_creduce_params& q = *reinterpret_cast<const spx_creduce_params*>(r.params.data());
      return q.dtype == SPX_DT_I32 ? spx_launch_creduce_i32(q, s, nl) : spx_launch_creduce(q, s, nl);
    }
    case SPX_K_GEMM:
      if (r.path == 4) return spx_launch_gemm_i32(*reinterpret_cast<const spx_gemm_params*>(r.params.data()), s, nl);
      if (r.path == 3) return spx_gemm_h3_launch(r.h3, s, nl);
      if (r.path == 1) return spx_gemm_tc_launch(r.tc, s, nl);
      return spx_launch_gemm_simt(*reinterpret_cast<const spx_gemm_params*>(r.params.data()), s, nl);
    case SPX_K_NCCL: return run_nccl(*reinterpret_cast<const spx_nccl_params*>(r.params.data()), s);
    case SPX_K_PEER: return spx_launch_peer(*reinterpret_cast<const spx_peer_params*>(r.params.data()), s, nl);
    case SPX_K_COPY: {
      const spx_copy_params& c = *reinterpret_cast<const spx_copy_params*>(r.params.data());
      if (!c.bytes) return 0;
      if (c.dir == 0)
        SPX_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(c.dev), reinterpret_cast<const void*>(c.host), c.bytes,
                                 cudaMemcpyHostToDevice, s));
      else if (c.dir == 1)
        SPX_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(c.host), reinterpret_cast<const void*>(c.dev), c.bytes,
                                 cudaMemcpyDeviceToHost, s));
      else   // 2: device -> device, `host` holds the (possibly peer-mapped) source
        SPX_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(c.dev), reinterpret_cast<const void*>(c.host), c.bytes,
                                 cudaMemcpyDeviceToDevice, s));
      cudaStreamCaptureStatus st;
      SPX_CUDA(cudaStreamIsCapturing(s, &st));
      if (c.dir != 2 && st == cudaStreamCaptureStatusActive) {
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        SPX_CUDA(cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd));
        r.node = nd ? deps[0] : nullptr;       // the memcpy node just captured
      }
      return 0;
    }
    case SPX_K_SPLIT:
      if (!r.batch_params.empty()) {
        std::vector<const spx_split_params*> ps;
        for (auto& q : r.batch_params) ps.push_back(&q);
        return spx_launch_split_batch(ps.data(), (int)ps.size(), s, nl);
      }
      return spx_launch_split(*reinterpret_cast<const spx_split_params*>(r.params.data()), s, nl);
  }
  return spx_set_error("unknown record kind %d", r.kind);
}



static size_t params_size(int kind) {
  switch (kind) {
    case SPX_K_EW: return sizeof(spx_ew_params);
    case SPX_K_REDUCE: return sizeof(spx_reduce_params);
    case SPX_K_GEMM: return sizeof(spx_gemm_params);
    case SPX_K_GATHER: return sizeof(spx_gather_params);
    case SPX_K_CREDUCE: return sizeof(spx_creduce_params);
    case SPX_K_NCCL: return sizeof(spx_nccl_params);
    case SPX_K_PEER: return sizeof(spx_peer_params);
    case SPX_K_SPLIT: return sizeof(spx_split_params);
    case SPX_K_COPY: return sizeof(spx_copy_params);
  }
  return 0;
}

extern "C" {

const char* spx_last_error(void) { return g_err; }
int spx_version(void) { return 1; }

int spx_params_size(int kind) { return (int)params_size(kind); }

int spx_device_init(int ordinal) {
  SPX_CUDA(cudaSetDevice(ordinal));
  cudaDeviceProp prop;
  SPX_CUDA(cudaGetDeviceProperties(&prop, ordinal));
  if (prop.major != 10) return spx_set_error("device %d is sm_%d%d; spindle_b200 needs sm_100 (B200)", ordinal, prop.major, prop.minor);
  g_num_sms = prop.multiProcessorCount;
  SPX_CUDA(cudaFree(0));
  return 0;
}

int spx_malloc(uint64_t bytes, uint64_t* out) {
  void* p = nullptr;
  SPX_CUDA(cudaMalloc(&p, bytes ? bytes : 256));
  *out = reinterpret_cast<uint64_t>(p);
  return 0;
}
int spx_free(uint64_t ptr) {
  SPX_CUDA(cudaFree(reinterpret_cast<void*>(ptr)));
  return 0;
}
int spx_mem_info(uint64_t* free_bytes, uint64_t* total_bytes) {
  size_t f = 0, t = 0;
  SPX_CUDA(cudaMemGetInfo(&f, &t));
  *free_bytes = f;
  *total_bytes = t;
  return 0;
}
int spx_memcpy_h2d(uint64_t dst, const void* src, uint64_t bytes, uint64_t stream) {
  SPX_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(dst), src, bytes, cudaMemcpyHostToDevice,
                           reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}
int spx_memcpy_d2h(void* dst, uint64_t src, uint64_t bytes, uint64_t stream) {
  SPX_CUDA(cudaMemcpyAsync(dst, reinterpret_cast<const void*>(src), bytes, cudaMemcpyDeviceToHost,
                           reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}
int spx_memcpy_d2d(uint64_t dst, uint64_t src, uint64_t bytes, uint64_t stream) {
  SPX_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(dst), reinterpret_cast<const void*>(src), bytes,
                           cudaMemcpyDeviceToDevice, reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}
int spx_memset(uint64_t dst, int value, uint64_t bytes, uint64_t stream) {
  SPX_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(dst), value, bytes, reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}
int spx_host_alloc(uint64_t bytes, void** out) {
  SPX_CUDA(cudaHostAlloc(out, bytes ? bytes : 16, cudaHostAllocDefault));
  return 0;
}
int spx_host_free(void* p) {
  SPX_CUDA(cudaFreeHost(p));
  return 0;
}
int spx_host_register(void* p, uint64_t bytes) {
  SPX_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  return 0;
}
int spx_host_unregister(void* p) {
  SPX_CUDA(cudaHostUnregister(p));
  return 0;
}
}  // extern "C"

// ---------------------------------------------------------------------------
// Staged host<->device copies for pageable host arrays (the drop-in call's
// inputs and results): a persistent pool of memcpy threads moves chunks
// between the user's memory and a ring of pinned buffers while the copy
// engine moves the previous chunk over PCIe -- pageable cudaMemcpy runs at
// ~11 GB/s H2D and ~5 GB/s D2H into fresh pages on this box, pinned DMA at
// ~55 GB/s and a 16-thread host memcpy at ~86 GB/s (tools/h2d_bench.py).
// ---------------------------------------------------------------------------
namespace {

class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 1; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
    n_ = n;
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // memcpy split over the pool (the calling thread takes part)
  void copy(void* dst, const void* src, size_t bytes) {
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(0);
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void part(int i) {
    const size_t per = ((bytes_ + n_ - 1) / n_ + 4095) & ~size_t(4095);
    const size_t o = per * i;
    if (o < bytes_) memcpy(dst_ + o, src_ + o, o + per > bytes_ ? bytes_ - o : per);
  }
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      part(i);
      {
        std::lock_guard<std::mutex> g(m_);
        --pending_;
      }
      done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
  int n_ = 1, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct Staging {
  static constexpr int R = 4;
  static constexpr size_t CHUNK = 32u << 20;
  void* buf[R] = {};
  cudaEvent_t ev[R] = {};
  CopyPool* pool = nullptr;
  std::mutex m;
};
Staging g_stage;

int staging_init() {
  if (g_stage.pool) return 0;
  for (int i = 0; i < Staging::R; ++i) {
    SPX_CUDA(cudaHostAlloc(&g_stage.buf[i], Staging::CHUNK, cudaHostAllocPortable));
    SPX_CUDA(cudaEventCreateWithFlags(&g_stage.ev[i], cudaEventDisableTiming));
  }
  int n = (int)std::thread::hardware_concurrency();
  const char* e = getenv("SPX_COPY_THREADS");
  if (e) n = atoi(e);
  if (n < 1) n = 1;
  if (n > 32) n = 32;
  g_stage.pool = new CopyPool(n);
  return 0;
}

}  // namespace

extern "C" {

int spx_h2d_staged(uint64_t dst, const void* src, uint64_t bytes, uint64_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (bytes < (4u << 20)) return spx_memcpy_h2d(dst, src, bytes, stream);
  std::lock_guard<std::mutex> g(g_stage.m);
  if (staging_init()) return -1;
  int k = 0;
  for (uint64_t o = 0; o < bytes; o += Staging::CHUNK, k = (k + 1) % Staging::R) {
    const uint64_t n = bytes - o < Staging::CHUNK ? bytes - o : Staging::CHUNK;
    SPX_CUDA(cudaEventSynchronize(g_stage.ev[k]));          // the slot's previous DMA is done
    g_stage.pool->copy(g_stage.buf[k], static_cast<const char*>(src) + o, n);
    SPX_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(dst + o), g_stage.buf[k], n, cudaMemcpyHostToDevice, s));
    SPX_CUDA(cudaEventRecord(g_stage.ev[k], s));
  }
  return 0;
}

int spx_d2h_staged(void* dst, uint64_t src, uint64_t bytes, uint64_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (bytes < (4u << 20)) {
    if (spx_memcpy_d2h(dst, src, bytes, stream)) return -1;
    SPX_CUDA(cudaStreamSynchronize(s));
    return 0;
  }
  std::lock_guard<std::mutex> g(g_stage.m);
  if (staging_init()) return -1;
  const uint64_t nchunks = (bytes + Staging::CHUNK - 1) / Staging::CHUNK;
  auto issue = [&](uint64_t c) -> int {
    const uint64_t o = c * Staging::CHUNK, n = bytes - o < Staging::CHUNK ? bytes - o : Staging::CHUNK;
    const int k = (int)(c % Staging::R);
    SPX_CUDA(cudaMemcpyAsync(g_stage.buf[k], reinterpret_cast<const void*>(src + o), n, cudaMemcpyDeviceToHost, s));
    SPX_CUDA(cudaEventRecord(g_stage.ev[k], s));
    return 0;
  };
  uint64_t issued = 0;
  for (; issued < nchunks && issued < (uint64_t)Staging::R; ++issued)
    if (issue(issued)) return -1;
  for (uint64_t c = 0; c < nchunks; ++c) {
    const uint64_t o = c * Staging::CHUNK, n = bytes - o < Staging::CHUNK ? bytes - o : Staging::CHUNK;
    const int k = (int)(c % Staging::R);
    SPX_CUDA(cudaEventSynchronize(g_stage.ev[k]));
    g_stage.pool->copy(static_cast<char*>(dst) + o, g_stage.buf[k], n);
    if (issued < nchunks && issue(issued++)) return -1;        // the slot is free again
  }
  return 0;
}

int spx_host_copy(void* dst, const void* src, uint64_t bytes, int threads) {
  if (threads <= 1 || bytes < (8u << 20)) {
    memcpy(dst, src, bytes);
    return 0;
  }
  std::vector<std::thread> ts;
  const uint64_t per = (bytes / threads + 4095) & ~uint64_t(4095);
  for (int t = 0; t < threads; ++t) {
    const uint64_t o = per * t;
    if (o >= bytes) break;
    const uint64_t n = o + per > bytes ? bytes - o : per;
    ts.emplace_back([=] { memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, n); });
  }
  for (auto& t : ts) t.join();
  return 0;
}
int spx_stream_create(uint64_t* out) {
  cudaStream_t s;
  SPX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = reinterpret_cast<uint64_t>(s);
  return 0;
}
int spx_stream_sync(uint64_t stream) {
  SPX_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}
int spx_stream_destroy(uint64_t stream) {
  SPX_CUDA(cudaStreamDestroy(reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}

int spx_ipc_get_handle(uint64_t ptr, uint8_t out_handle[64]) {
  cudaIpcMemHandle_t h;
  SPX_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(ptr)));
  memcpy(out_handle, &h, sizeof(h) < 64 ? sizeof(h) : 64);
  return 0;
}
int spx_ipc_open(const uint8_t handle[64], uint64_t* out_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h) < 64 ? sizeof(h) : 64);
  void* p = nullptr;
  SPX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *out_ptr = reinterpret_cast<uint64_t>(p);
  return 0;
}
int spx_ipc_close(uint64_t ptr) {
  SPX_CUDA(cudaIpcCloseMemHandle(reinterpret_cast<void*>(ptr)));
  return 0;
}

int spx_nccl_get_unique_id(uint8_t out_id[128]) {
  if (nccl_load()) return -1;
  nccl_uid_t id;
  SPX_NCCL(N.get_uid(&id));
  memcpy(out_id, id.internal, 128);
  return 0;
}
int spx_comm_init(const uint8_t id[128], int nranks, int rank, int* out_comm) {
  if (nccl_load()) return -1;
  nccl_uid_t uid;
  memcpy(uid.internal, id, 128);
  nccl_comm_t c = nullptr;
  SPX_NCCL(N.init_rank(&c, nranks, uid, rank));
  g_comms.push_back(c);
  *out_comm = (int)g_comms.size() - 1;
  return 0;
}
int spx_comm_destroy(int comm) {
  if (comm < 0 || comm >= (int)g_comms.size() || !g_comms[comm]) return 0;
  SPX_NCCL(N.destroy(g_comms[comm]));
  g_comms[comm] = nullptr;
  return 0;
}

int spx_comm_async_error(int comm, int* out) {
  *out = 0;
  if (comm < 0 || comm >= (int)g_comms.size() || !g_comms[comm]) return 0;
  int e = 0;
  SPX_NCCL(N.async_error(g_comms[comm], &e));
  *out = e;
  return 0;
}

int spx_comm_abort(int comm) {
  if (comm < 0 || comm >= (int)g_comms.size() || !g_comms[comm]) return 0;
  N.abort(g_comms[comm]);
  g_comms[comm] = nullptr;
  return 0;
}

int spx_peer_error(int* out);

// Wait for `stream` while watching for failures: an NCCL asynchronous error on
// any live communicator (ncclCommGetAsyncError; the communicators are then
// aborted so their kernels return), a peer-collective barrier that gave up
// (spx_peer_error), or no completion within timeout_s (0: none).  Returns 0
// when the stream completed cleanly.
int spx_stream_sync_watch(uint64_t stream, double timeout_s) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const auto t0 = std::chrono::steady_clock::now();
  for (int it = 0;; ++it) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return spx_set_error("stream: %s", cudaGetErrorString(q));
    if (N.h && (it & 15) == 0) {
      for (size_t c = 0; c < g_comms.size(); ++c) {
        if (!g_comms[c]) continue;
        int e = 0;
        if (N.async_error(g_comms[c], &e) == 0 && e != 0 && e != 7 /* ncclInProgress */) {
          for (size_t k = 0; k < g_comms.size(); ++k) spx_comm_abort((int)k);
          return spx_set_error("NCCL asynchronous error %d (%s) on communicator %zu; communicators aborted", e,
                               N.errstr(e), c);
        }
      }
    }
    int pe = 0;
    spx_peer_error(&pe);
    if (pe) return spx_set_error("peer collective barrier (phase %d) timed out: a member never arrived", pe - 1);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_s > 0 && el > timeout_s) return spx_set_error("stream did not complete within %.0f s", timeout_s);
    std::this_thread::sleep_for(std::chrono::microseconds(it < 100 ? 20 : 500));
  }
  int pe = 0;
  spx_peer_error(&pe);
  if (pe) return spx_set_error("peer collective barrier (phase %d) timed out: a member never arrived", pe - 1);
  return 0;
}

int spx_plan_create(uint64_t* out) {
  *out = reinterpret_cast<uint64_t>(new Plan());
  return 0;
}

int spx_plan_add(uint64_t plan, int kind, const void* params, uint64_t bytes) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (P->finalized) return spx_set_error("plan already finalized");
  const size_t want = params_size(kind);
  if (!want) return spx_set_error("unknown record kind %d", kind);
  if (bytes != want) return spx_set_error("record kind %d: %llu bytes, ABI says %zu", kind, (unsigned long long)bytes, want);
  Record r;
  r.kind = kind;
  r.path = 0;
  r.params.assign(static_cast<const uint8_t*>(params), static_cast<const uint8_t*>(params) + bytes);
  if (kind == SPX_K_EW) {
    const char* e = getenv("SPX_EW_STATIC");
    if (!(e && e[0] == '0') && reinterpret_cast<const spx_ew_params*>(r.params.data())->dtype == SPX_DT_F32)
      r.path = 1 + spx_ew_static_match(*reinterpret_cast<const spx_ew_params*>(r.params.data()));
    const spx_ew_params& q = *reinterpret_cast<const spx_ew_params*>(r.params.data());
    if (r.path == 0 && q.dtype == SPX_DT_F32 && spx_ew_jit_enabled()) {
      if (spx_ew_jit_prepare(q, &r.jit)) return -1;
      r.path = -3;
    }
  }
  if (kind == SPX_K_GEMM && reinterpret_cast<const spx_gemm_params*>(r.params.data())->dtype == SPX_DT_I32) {
    const spx_gemm_params& g = *reinterpret_cast<const spx_gemm_params*>(r.params.data());
    if (g.splits > 1 || g.epi != SPX_EPI_NONE || g.h3_shared || (g.path != 0 && g.path != 2))
      return spx_set_error("gemm %dx%dx%d: int32 GEMMs run on the SIMT path only", g.M, g.N, g.K);
    r.path = 4;
  } else if (kind == SPX_K_GEMM) {
    const spx_gemm_params& g = *reinterpret_cast<const spx_gemm_params*>(r.params.data());
    const bool tc_ok = spx_gemm_tc_supported(g);
    if (g.path == 1 && !tc_ok) return spx_set_error("gemm %dx%dx%d: tcgen05 path requested but operands unsupported", g.M, g.N, g.K);
    if (g.h3_shared && g.path != 3) return spx_set_error("gemm %dx%dx%d: shared fp16 pieces need path 3", g.M, g.N, g.K);
    if (g.path == 3) {
      if (!spx_gemm_h3_supported(g))
        return spx_set_error("gemm %dx%dx%d: block-scaled fp16 path requested but unsupported", g.M, g.N, g.K);
      r.path = 3;
    } else {
      r.path = (g.path == 2 || (g.path == 0 && !tc_ok)) ? 2 : 1;
      if (g.path == 0 && r.path == 1 && h3_default() && spx_gemm_h3_supported(g)) r.path = 3;
    }
    if (g.splits > 1 && r.path != 1) return spx_set_error("gemm %dx%dx%d: split-K needs the tcgen05 path", g.M, g.N, g.K);
    if (g.epi != SPX_EPI_NONE && r.path != 1) return spx_set_error("gemm %dx%dx%d: fused epilogue needs the tcgen05 path", g.M, g.N, g.K);
  }
  r.flops = record_flops(r);
  P->recs.push_back(std::move(r));
  return 0;
}

int spx_plan_finalize(uint64_t plan) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  int64_t h3need[SPX_SIDE_STREAMS + 1] = {};
  for (auto& r : P->recs) {
    if (r.kind == SPX_K_GEMM && r.path == 1 && !r.tc) {
      if (spx_gemm_tc_prepare(*reinterpret_cast<const spx_gemm_params*>(r.params.data()), &r.tc)) return -1;
    }
    if (r.kind == SPX_K_GEMM && r.path == 3 && !r.h3) {
      if (spx_gemm_h3_prepare(*reinterpret_cast<const spx_gemm_params*>(r.params.data()), &r.h3)) return -1;
      const int64_t b = spx_gemm_h3_ws_bytes(r.h3);
      if (b > h3need[r.stream]) h3need[r.stream] = b;
    }
    if (r.signal && !r.done) SPX_CUDA(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
  }
  // elementwise record + the split of its output right after it on the same
  // stream: one launch (ew_static.cu ew_static_split_kernel)
  static int fuse = -1;
  if (fuse < 0) {
    const char* e = getenv("SPX_EW_SPLIT_FUSE");
    fuse = e ? atoi(e) != 0 : 1;
  }
  const char* jse = getenv("SPX_EW_JIT_SPLIT");
  const bool jit_split = !(jse && atoi(jse) == 0);
  const char* poe = getenv("SPX_PIECES_ONLY");
  const bool pieces_only = !(poe && atoi(poe) == 0);
  for (size_t i = 0; fuse && i + 1 < P->recs.size(); ++i) {
    Record &a = P->recs[i], &b = P->recs[i + 1];
    const bool jit = a.path == -3 && a.jit && jit_split;
    if (a.kind != SPX_K_EW || (a.path <= 0 && !jit) || b.kind != SPX_K_SPLIT || a.stream != b.stream ||
        !b.waits.empty() || a.fused_split >= 0)
      continue;
    const int j = spx_ew_split_match(*reinterpret_cast<const spx_ew_params*>(a.params.data()),
                                     *reinterpret_cast<const spx_split_params*>(b.params.data()));
    if (j < 0) continue;
    if (jit) {
      // the generated kernel with the split's cluster structure around it
      const spx_split_params& sp = *reinterpret_cast<const spx_split_params*>(b.params.data());
      const int skip = pieces_only && (sp.flags & SPX_SPLIT_PIECES_ONLY) ? 1 : 0;
      if (spx_ew_jit_split_prepare(*reinterpret_cast<const spx_ew_params*>(a.params.data()), sp, j, skip,
                                   &a.jit_split)) {
        g_err[0] = 0;
        continue;                 // not fusable (e.g. >= 2^31 elements): the split runs on its own
      }
    }
    a.fused_split = (int)(i + 1);
    a.split_out = j;
    a.split_params = b.params;
    b.fused = true;
    b.path = -1;                 // reported by spx_plan_record_info: runs inside record i
  }
  // consecutive standalone splits on one stream (the hoisted splits of the
  // weights, ...): one batched launch at the first (gemm_h3.cu split_h16_batch_kernel)
  const char* be = getenv("SPX_SPLIT_BATCH");
  const int batch = be ? atoi(be) != 0 : 1;
  // SPX_SPLIT_BATCH_FIRST=k: the first batch of a stream holds only k splits,
  // so the step's first GEMM does not wait for every weight's split (0.29 ms
  // in the eager C2 N=1 timeline); measured neutral under graph replay (C2
  // N=1 558.7k, C4 84.7k), so off by default
  const char* bfe = getenv("SPX_SPLIT_BATCH_FIRST");
  const int first_cap = bfe ? atoi(bfe) : 0;
  bool first_done[SPX_SIDE_STREAMS + 1] = {};
  for (size_t i = 0; batch && i < P->recs.size(); ++i) {
    Record& a = P->recs[i];
    if (a.kind != SPX_K_SPLIT || a.fused) continue;
    const int cap = (!first_done[a.stream] && first_cap > 0) ? first_cap : spx_split_batch_max();
    first_done[a.stream] = true;
    size_t j = i + 1;
    for (; j < P->recs.size() && (int)a.batch.size() + 1 < cap; ++j) {
      Record& b = P->recs[j];
      if (b.kind != SPX_K_SPLIT || b.fused || b.stream != a.stream || !b.waits.empty()) break;
      a.batch.push_back((int)j);
      b.fused = true;
      b.path = -2;               // reported by spx_plan_record_info: runs inside the batch of record i
    }
    if (!a.batch.empty()) {
      a.path = 2;
      a.batch_params.push_back(*reinterpret_cast<const spx_split_params*>(a.params.data()));
      for (int k : a.batch) a.batch_params.push_back(*reinterpret_cast<const spx_split_params*>(P->recs[k].params.data()));
    }
    i = j - 1;
  }
  for (int k = 0; k <= SPX_SIDE_STREAMS; ++k)
    if (h3need[k] && !P->h3ws[k]) SPX_CUDA(cudaMalloc(&P->h3ws[k], (size_t)h3need[k]));
  for (auto& r : P->recs)
    if (r.h3 && spx_gemm_h3_bind(r.h3, reinterpret_cast<uint64_t>(P->h3ws[r.stream]))) return -1;
  if (P->two_streams) {
    int lo = 0, hi = 0;
    SPX_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int k = 1; k <= SPX_SIDE_STREAMS; ++k) {
      if (!P->used[k]) continue;
      // collectives (and the legacy single side stream) first
      SPX_CUDA(cudaStreamCreateWithPriority(&P->side[k], cudaStreamNonBlocking, k == 2 || k == 1 ? hi : lo));
      SPX_CUDA(cudaEventCreateWithFlags(&P->join[k], cudaEventDisableTiming));
    }
    SPX_CUDA(cudaEventCreateWithFlags(&P->fork, cudaEventDisableTiming));
  }
  P->finalized = true;
  return 0;
}

// Issue every record: main-stream records on `s`, side-stream records on the
// plan's side stream, cross-stream order through events (fork at the start,
// join at the end, so the whole plan is one unit on `s` -- also under capture).
static int issue_all(Plan* P, cudaStream_t s, int* nl, spx_exec_stats* t) {
  *t = spx_exec_stats{};
  t->runs = 1;
  if (!P->two_streams) {
    for (auto& r : P->recs) {
      if (run_record(r, s, nl)) return -1;
      tally_record(r, t);
    }
    t->launches = *nl;
    return 0;
  }
  SPX_CUDA(cudaEventRecord(P->fork, s));
  for (int k = 1; k <= SPX_SIDE_STREAMS; ++k)
    if (P->used[k]) SPX_CUDA(cudaStreamWaitEvent(P->side[k], P->fork, 0));
  for (auto& r : P->recs) {
    cudaStream_t rs = r.stream ? P->side[r.stream] : s;
    for (int w : r.waits) SPX_CUDA(cudaStreamWaitEvent(rs, P->recs[w].done, 0));
    if (run_record(r, rs, nl)) return -1;
    tally_record(r, t);
    if (r.signal) SPX_CUDA(cudaEventRecord(r.done, rs));
  }
  for (int k = 1; k <= SPX_SIDE_STREAMS; ++k) {
    if (!P->used[k]) continue;
    SPX_CUDA(cudaEventRecord(P->join[k], P->side[k]));
    SPX_CUDA(cudaStreamWaitEvent(s, P->join[k], 0));
  }
  t->launches = *nl;
  return 0;
}

static void stats_add(spx_exec_stats* a, const spx_exec_stats& b) {
  a->runs += b.runs;
  for (int k = 0; k < 4; ++k) a->coll[k] += b.coll[k];
  a->flops += b.flops;
  a->launches += b.launches;
}

int spx_plan_set_sched(uint64_t plan, int index, int stream, const int* waits, int n_waits) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (P->finalized) return spx_set_error("plan already finalized");
  if (index < 0 || index >= (int)P->recs.size()) return spx_set_error("record index out of range");
  Record& r = P->recs[index];
  if (stream < 0 || stream > SPX_SIDE_STREAMS) return spx_set_error("stream %d out of range", stream);
  r.stream = stream;
  r.waits.clear();
  for (int i = 0; i < n_waits; ++i) {
    const int w = waits[i];
    if (w < 0 || w >= index) return spx_set_error("record %d waits for %d: not an earlier record", index, w);
    r.waits.push_back(w);
    P->recs[w].signal = true;
  }
  if (r.stream) {
    P->two_streams = true;
    P->used[r.stream] = true;
  }
  return 0;
}

int spx_plan_run(uint64_t plan, uint64_t stream) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (!P->finalized && spx_plan_finalize(plan)) return -1;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int nl = 0;
  spx_exec_stats t;
  if (issue_all(P, s, &nl, &t)) return -1;
  stats_add(&P->stats, t);
  P->launches = nl;
  return 0;
}

int spx_plan_capture(uint64_t plan, uint64_t stream) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (!P->finalized && spx_plan_finalize(plan)) return -1;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (P->exec) { cudaGraphExecDestroy(P->exec); P->exec = nullptr; }
  if (P->graph) { cudaGraphDestroy(P->graph); P->graph = nullptr; }
  SPX_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int nl = 0;
  if (issue_all(P, s, &nl, &P->graph_tally)) {
    cudaGraph_t g;
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    return -1;
  }
  SPX_CUDA(cudaStreamEndCapture(s, &P->graph));
  SPX_CUDA(cudaGraphInstantiate(&P->exec, P->graph, 0));
  P->launches = nl;
  return 0;
}

int spx_plan_replay(uint64_t plan, uint64_t stream) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (!P->exec) return spx_set_error("plan has no captured graph");
  SPX_CUDA(cudaGraphLaunch(P->exec, reinterpret_cast<cudaStream_t>(stream)));
  stats_add(&P->stats, P->graph_tally);
  return 0;
}

int spx_plan_tag(uint64_t plan, int index, int tag) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (index < 0 || index >= (int)P->recs.size()) return spx_set_error("record index out of range");
  const int c = tag & SPX_TAG_COLL_MASK;
  if (c > 4 || (tag & ~(SPX_TAG_COLL_MASK | SPX_TAG_INTERNAL))) return spx_set_error("bad record tag %#x", tag);
  P->recs[index].tag = tag;
  return 0;
}

int spx_h3_range_events(uint32_t* out, int reset) {
  uint32_t a = 0, b = 0;
  if (spx_h3_range_split(&a, reset) || spx_h3_range_ew(&b, reset)) return -1;
  *out = a + b;
  return 0;
}

int spx_plan_set_host(uint64_t plan, int index, uint64_t host) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (index < 0 || index >= (int)P->recs.size()) return spx_set_error("record index out of range");
  Record& r = P->recs[index];
  if (r.kind != SPX_K_COPY) return spx_set_error("record %d is not a copy", index);
  spx_copy_params& c = *reinterpret_cast<spx_copy_params*>(r.params.data());
  c.host = host;
  if (P->exec && r.node && c.bytes) {
    if (c.dir == 0)
      SPX_CUDA(cudaGraphExecMemcpyNodeSetParams1D(P->exec, r.node, reinterpret_cast<void*>(c.dev),
                                                  reinterpret_cast<const void*>(c.host), c.bytes, cudaMemcpyHostToDevice));
    else
      SPX_CUDA(cudaGraphExecMemcpyNodeSetParams1D(P->exec, r.node, reinterpret_cast<void*>(c.host),
                                                  reinterpret_cast<const void*>(c.dev), c.bytes, cudaMemcpyDeviceToHost));
  }
  return 0;
}

int spx_plan_exec_stats(uint64_t plan, spx_exec_stats* out) {
  *out = reinterpret_cast<Plan*>(plan)->stats;
  return 0;
}

int spx_plan_reset_stats(uint64_t plan) {
  reinterpret_cast<Plan*>(plan)->stats = spx_exec_stats{};
  return 0;
}

int spx_plan_launch_count(uint64_t plan) { return reinterpret_cast<Plan*>(plan)->launches; }

int spx_plan_record_info(uint64_t plan, int index, int* kind, int* path) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (index < 0 || index >= (int)P->recs.size()) return spx_set_error("record index out of range");
  *kind = P->recs[index].kind;
  *path = P->recs[index].path;
  return 0;
}

int spx_plan_destroy(uint64_t plan) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (P->exec) cudaGraphExecDestroy(P->exec);
  if (P->graph) cudaGraphDestroy(P->graph);
  for (auto& r : P->recs) {
    if (r.tc) spx_gemm_tc_free(r.tc);
    if (r.h3) spx_gemm_h3_free(r.h3);
    if (r.jit) spx_ew_jit_free(r.jit);
    if (r.jit_split) spx_ew_jit_free(r.jit_split);
    if (r.done) cudaEventDestroy(r.done);
  }
  for (int k = 1; k <= SPX_SIDE_STREAMS; ++k) {
    if (P->side[k]) cudaStreamDestroy(P->side[k]);
    if (P->join[k]) cudaEventDestroy(P->join[k]);
  }
  if (P->fork) cudaEventDestroy(P->fork);
  for (int k = 0; k <= SPX_SIDE_STREAMS; ++k)
    if (P->h3ws[k]) cudaFree(P->h3ws[k]);
  delete P;
  return 0;
}

int spx_event_create(uint64_t* out) {
  cudaEvent_t e;
  SPX_CUDA(cudaEventCreate(&e));
  *out = reinterpret_cast<uint64_t>(e);
  return 0;
}
int spx_event_record(uint64_t ev, uint64_t stream) {
  SPX_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}
int spx_stream_wait_event(uint64_t stream, uint64_t ev) {
  SPX_CUDA(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<cudaEvent_t>(ev), 0));
  return 0;
}
int spx_event_elapsed_ms(uint64_t a, uint64_t b, float* out) {
  SPX_CUDA(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(b)));
  SPX_CUDA(cudaEventElapsedTime(out, reinterpret_cast<cudaEvent_t>(a), reinterpret_cast<cudaEvent_t>(b)));
  return 0;
}
int spx_event_destroy(uint64_t ev) {
  SPX_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev)));
  return 0;
}

// Timeline of one multi-stream run (dev tool, tools/timeline.py): every record
// issued on its own stream as in issue_all, with an event after its waits
// (`ready`: the stream reached it and its cross-stream dependencies were met)
// and one after it (`end`), both in ms from the start of the run.  The host
// enqueues the whole run behind a hold kernel, so the times carry no host
// launch gaps (like a graph replay).
int spx_plan_trace(uint64_t plan, uint64_t stream, float* ready_ms, float* end_ms, int n) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (!P->finalized && spx_plan_finalize(plan)) return -1;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nr = (int)P->recs.size();
  std::vector<cudaEvent_t> ev(2 * nr + 1);
  for (auto& e : ev) SPX_CUDA(cudaEventCreate(&e));
  long long hold = 40000LL * nr + 2000000LL;
  if (hold > 400000000LL) hold = 400000000LL;
  hold_stream_kernel<<<1, 32, 0, s>>>(hold);
  SPX_CUDA(cudaGetLastError());
  SPX_CUDA(cudaEventRecord(ev[0], s));
  if (P->two_streams) {
    SPX_CUDA(cudaEventRecord(P->fork, s));
    for (int k = 1; k <= SPX_SIDE_STREAMS; ++k)
      if (P->used[k]) SPX_CUDA(cudaStreamWaitEvent(P->side[k], P->fork, 0));
  }
  int nl = 0;
  spx_exec_stats t = {};
  t.runs = 1;
  for (int i = 0; i < nr; ++i) {
    Record& r = P->recs[i];
    cudaStream_t rs = (P->two_streams && r.stream) ? P->side[r.stream] : s;
    if (P->two_streams)
      for (int w : r.waits) SPX_CUDA(cudaStreamWaitEvent(rs, P->recs[w].done, 0));
    SPX_CUDA(cudaEventRecord(ev[1 + 2 * i], rs));
    if (run_record(r, rs, &nl)) return -1;
    tally_record(r, &t);
    SPX_CUDA(cudaEventRecord(ev[2 + 2 * i], rs));
    if (P->two_streams && r.signal) SPX_CUDA(cudaEventRecord(r.done, rs));
  }
  if (P->two_streams) {
    for (int k = 1; k <= SPX_SIDE_STREAMS; ++k) {
      if (!P->used[k]) continue;
      SPX_CUDA(cudaEventRecord(P->join[k], P->side[k]));
      SPX_CUDA(cudaStreamWaitEvent(s, P->join[k], 0));
    }
  }
  t.launches = nl;
  stats_add(&P->stats, t);
  SPX_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < nr && i < n; ++i) {
    SPX_CUDA(cudaEventElapsedTime(&ready_ms[i], ev[0], ev[1 + 2 * i]));
    SPX_CUDA(cudaEventElapsedTime(&end_ms[i], ev[0], ev[2 + 2 * i]));
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return 0;
}

int spx_plan_profile(uint64_t plan, uint64_t stream, float* out_ms, int n) {
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (!P->finalized && spx_plan_finalize(plan)) return -1;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nr = (int)P->recs.size();
  std::vector<cudaEvent_t> ev(nr + 1);
  for (auto& e : ev) SPX_CUDA(cudaEventCreate(&e));
  // hold the stream while the host enqueues every record and event, so the
  // per-record times are device execution back to back (no host launch gaps)
  long long hold = 20000LL * nr + 1000000LL;
  if (hold > 200000000LL) hold = 200000000LL;
  hold_stream_kernel<<<1, 32, 0, s>>>(hold);
  SPX_CUDA(cudaGetLastError());
  SPX_CUDA(cudaEventRecord(ev[0], s));
  int nl = 0;
  spx_exec_stats t = {};
  t.runs = 1;
  for (int i = 0; i < nr; ++i) {
    if (run_record(P->recs[i], s, &nl)) return -1;
    tally_record(P->recs[i], &t);
    SPX_CUDA(cudaEventRecord(ev[i + 1], s));
  }
  t.launches = nl;
  stats_add(&P->stats, t);
  SPX_CUDA(cudaEventSynchronize(ev[nr]));
  for (int i = 0; i < nr && i < n; ++i) SPX_CUDA(cudaEventElapsedTime(&out_ms[i], ev[i], ev[i + 1]));
  for (auto& e : ev) cudaEventDestroy(e);
  return 0;
}

}  // extern "C"
