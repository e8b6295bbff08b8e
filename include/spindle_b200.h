/*
 * spindle_b200 -- C-ABI of the B200-native partitioned-program evaluator.
 *
 * This is the drop-in boundary below the reference's `spmd_interpret`
 * (/root/reference/pkg/src/spindle/spmd_interp.py:157-197).  The reference's
 * per-op numpy kernels (`_eval_op`, interp.py:35-75) and numpy collective
 * emulation (`_run_collective`, spmd_interp.py:74-123) are replaced by the
 * launchers behind `spx_plan_*`; the host mirror of the reference interface
 * (paper_2401_11202_b200/evaluator.py) compiles a localized module + its
 * ShardingSpec into a plan of the records declared here and drives it.
 *
 * Conventions
 *   - every function returns 0 on success, a negative code on failure; the
 *     message is available from spx_last_error() (thread-local);
 *   - pointers are plain device addresses (uint64_t), sizes are in ELEMENTS
 *     of 4 bytes unless a name says _bytes.  No torch types cross the ABI;
 *   - "virtual devices": one process may host V mesh devices on one GPU; their
 *     buffers live at   base + d * dev_stride   (bytes) for d in [0, V), so
 *     every record below applies to all V devices in ONE launch.
 *
 * Reference interfaces replaced (file:line in /root/reference/pkg/src/spindle):
 *   SPX_K_EW       interp.py:39-52,58-67  constant/add/mul/neg/exp/transpose/
 *                                         broadcast/reshape/tag (fused chains)
 *   SPX_K_REDUCE   interp.py:53-55        reduce sum|max over any dims
 *   SPX_K_GEMM     interp.py:43-44        matmul (rank-2), operand transposes
 *                                         folded (interp.py:51-52)
 *   SPX_K_GATHER   spmd_interp.py:76-91,105-122  all_slice / all_gather /
 *                                         all_to_all data movement
 *   SPX_K_CREDUCE  spmd_interp.py:66-71,92-104   all_reduce / reduce_scatter
 *                                         (left fold in group order)
 *   SPX_K_NCCL     same collectives across processes (one GPU per mesh device)
 *   SPX_K_SPLIT    (no reference counterpart) fp32 operand -> block-scaled fp16
 *                  pieces feeding the 3xFP16 matmul path
 */
#ifndef SPINDLE_B200_H
#define SPINDLE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPX_MAX_RANK 6
#define SPX_MAX_IN 8
#define SPX_MAX_OUT 4
#define SPX_MAX_PROG 28

/* ---- elementwise expression programs (bytecode) ------------------------ */
enum spx_opcode {
  SPX_OP_MOV = 0,   /* t = a                  */
  SPX_OP_ADD = 1,   /* t = a + b   (IEEE fp32, round-to-nearest, no FMA) */
  SPX_OP_MUL = 2,   /* t = a * b               */
  SPX_OP_NEG = 3,   /* t = -a                  */
  SPX_OP_EXP = 4,   /* t = exp(a)              */
  SPX_OP_MAX = 5,   /* t = maximum(a, b)  (NaN-propagating, like np.maximum) */
  SPX_OP_IMM = 6,   /* t = imm[i]              */
  SPX_OP_ADDI = 7,  /* t = a + imm[i]  (constant operand on the right)  */
  SPX_OP_MULI = 8,  /* t = a * imm[i]          */
  SPX_OP_IADD = 9,  /* t = imm[i] + a  (constant operand on the left)   */
  SPX_OP_IMUL = 10  /* t = imm[i] * a          */
};

/* Register machine: SPX_NREG value slots; input view j is preloaded into slot
 * j, instruction i computes op(slot a, slot b [, imm[i]]) into slot dst.  The
 * host allocates slots by liveness (paper_2401_11202_b200/plan.py). */
#define SPX_NREG 12

typedef struct {
  int32_t op, a, b, dst;
} spx_insn;

typedef struct {
  int64_t off;                    /* element offset from the device base      */
  int64_t stride[SPX_MAX_RANK];   /* element strides per output dim (0 = bcast) */
} spx_view;

typedef struct {
  uint64_t base;                  /* device 0 arena base address              */
  int64_t dev_stride;             /* bytes between virtual devices            */
  int32_t ndev, rank, n_in, n_out, n_prog, vec;  /* vec: 1 = float4 fast path */
  int32_t dtype, dtype_pad;       /* SPX_DT_F32 / SPX_DT_I32 (imm[] then holds int32 bits) */
  int64_t dims[SPX_MAX_RANK];     /* logical output shape (row-major)         */
  int64_t numel;
  spx_view in[SPX_MAX_IN];
  int64_t out_off[SPX_MAX_OUT];   /* outputs are contiguous row-major          */
  int32_t out_reg[SPX_MAX_OUT];   /* which slot each output stores            */
  spx_insn prog[SPX_MAX_PROG];
  float imm[SPX_MAX_PROG];
} spx_ew_params;

/* Arithmetic type of a record (the reference computes in np.result_type of the
 * inputs, spmd_interp.py:173; the IR's element kinds are f32 and i32,
 * ir.py:14).  i32 arithmetic wraps modulo 2^32 like numpy's int32 ufuncs. */
enum spx_dtype { SPX_DT_F32 = 0, SPX_DT_I32 = 1 };

/* ---- reductions ---------------------------------------------------------- */
typedef struct {
  spx_ew_params x;                /* the reduced operand as an expression over
                                     the INPUT shape (out_reg[0] = value)      */
  int32_t monoid;                 /* 0 sum, 1 max                              */
  int32_t n_kept, n_red;          /* x.dims = kept (n_kept dims) ++ reduced      */
  int32_t mode;                   /* 0 ROW / 1 COL (2-D, x.vec = float4 along the
                                     fast dim), 2 GEN (any rank), 3 OUT (few
                                     reduced elements; 4 outputs per thread)   */
  int64_t kept_dims[SPX_MAX_RANK], kept_stride[SPX_MAX_RANK]; /* in input index space */
  int64_t red_dims[SPX_MAX_RANK], red_stride[SPX_MAX_RANK];
  int64_t n_out, n_red_elems;
  int64_t out_off;                /* contiguous output                         */
  int64_t scratch_off;            /* arena scratch for partials (elements)     */
} spx_reduce_params;

/* ---- matmul -------------------------------------------------------------- */
typedef struct {
  uint64_t base;
  int64_t dev_stride;             /* bytes */
  int32_t ndev, M, N, K;
  int64_t a_off, b_off, c_off;    /* elements from device base */
  int64_t lda, ldb, ldc;          /* row pitch (elements) of the STORED arrays */
  int32_t a_mn_major;             /* 0: A stored [M][K]; 1: A stored [K][M]    */
  int32_t b_k_major;              /* 0: B stored [K][N]; 1: B stored [N][K]    */
  int32_t path;                   /* 0 auto, 1 tcgen05 3xTF32, 2 SIMT fp32     */
  int32_t promote;                /* k-blocks per TMEM chunk (0 = default 4)     */
  int32_t reserve_sms;            /* SMs left free for concurrent collectives    */
  int32_t splits;                 /* split-K: >1 writes [splits][M][ldc] partials at c_off
                                     (sk_mode 0), or reduces them in the kernel (sk_mode 1) */
  /* Fused epilogue (tcgen05 path, splits == 1): the elementwise consumer of
   * C = A.B computed on the accumulator rows before they leave the SM, with
   * the same IEEE operations (and order) as the unfused kernel:
   *   SPX_EPI_NONE      out0 = C (at c_off / ldc)
   *   SPX_EPI_ADD       out0 = X0 + C                      (residual add)
   *   SPX_EPI_SQUARE    out0 = C, out1 = C * C              (square activation)
   *   SPX_EPI_MULSCALE  out0 = C * (X0 * imm0)              (its backward)
   *   SPX_EPI_MOMENTUM  out0 = X0 * imm0 + C,               (momentum SGD:
   *                     out1 = X1 + -(out0 * imm1)           m' then p')
   * X / out views: element offset from the device base + row pitch; columns
   * contiguous. */
  int32_t epi, epi_pad;
  int64_t epi_in_off[2], epi_in_ld[2];
  int64_t epi_out_off[2], epi_out_ld[2];
  float epi_imm[2];
  /* In-kernel split-K (sk_mode 1, tcgen05 path): the CTAs of split s > 0
   * store their partial tile into a workspace [splits-1][M][N] at ws_off and
   * count it into a per-(tile, row slice) flag at flag_off (uint32, zero
   * between launches); the split-0 CTAs wait for their flags, fold the
   * partials in split order (deterministic) and write C.  Every work unit
   * must be co-resident: tiles x splits x 2 <= SM count. */
  int32_t sk_mode, sk_pad;
  int64_t ws_off, flag_off;
  /* path 3 (block-scaled 3xFP16, splits == 1, no epilogue): with h3_shared the
   * operands' fp16 pieces and scales were written by SPX_K_SPLIT records into
   * the arena (offsets in elements from the device base; one split serves
   * every GEMM that reads the same tensor view); without it the record splits
   * its operands itself into a per-stream workspace. */
  int32_t h3_shared;
  int32_t h3_splitk;              /* path 3 split-K of few-tile GEMMs: <= 1 off (default), n = at most n splits */
  int64_t h3_a_off, h3_a_scl, h3_b_off, h3_b_scl;
  int32_t dtype, dtype_pad;       /* SPX_DT_I32: wrapping int32 GEMM (SIMT) */
} spx_gemm_params;

/* ---- operand split for the block-scaled 3xFP16 GEMM ------------------------
 * fp32 view [rows][cols] (row pitch ld) -> per 128 x 128 block a power-of-two
 * scale s (max |x| * s in [2^14, 2^15)), fp16 pieces hi = rn(x s),
 * lo = rn(x s - hi) at dst_off: [2][rows][pitch] halves, and 1/s per block at
 * scl_off: [ceil(rows/128)][ceil(cols/128)] fp32. */
typedef struct {
  uint64_t base;
  int64_t dev_stride;             /* bytes */
  int32_t ndev, rows, cols;
  int32_t flags;                  /* SPX_SPLIT_PIECES_ONLY: when this split runs inside the elementwise
                                     launch producing its source, that launch need not store the fp32
                                     source (every reader takes the pieces) */
  int64_t src_off, ld;            /* elements */
  int64_t dst_off, pitch;         /* pieces: elements from the device base; pitch in halves (multiple of 8) */
  int64_t scl_off;                /* elements */
} spx_split_params;

#define SPX_SPLIT_PIECES_ONLY 1

/* 128 x 128 blocks split since the last reset whose maximum |x| lay outside
 * [2^-45, 2^75], where the power-of-two scale is clamped to 2^+-60 and the
 * block's small elements keep only ~2^-40-of-the-maximum accuracy (the host
 * warns, or raises with SPX_STRICT_RANGE=1) */
int spx_h3_range_events(uint32_t* out, int reset);

enum spx_epilogue { SPX_EPI_NONE = 0, SPX_EPI_ADD = 1, SPX_EPI_SQUARE = 2, SPX_EPI_MULSCALE = 3,
                    SPX_EPI_MOMENTUM = 4 };

/* ---- collectives over co-located virtual devices ------------------------- */
/* gather-style (all_slice, all_gather, all_to_all, relayouts):
 *   out[d][l] = src[table[d * n_combo + combo(l)]] [ base_off[d] + sum_k (l_k % ext_k) * sstride_k ]
 * where combo(l) = sum_k (l_k / ext_k) * cmul_k.  Tables are device arrays. */
typedef struct {
  int32_t ndev, rank, n_combo, pad;
  int64_t dims[SPX_MAX_RANK];     /* output local shape */
  int64_t ext[SPX_MAX_RANK];      /* chunk extent per dim (== dims if not split) */
  int64_t cmul[SPX_MAX_RANK];
  int64_t sstride[SPX_MAX_RANK];  /* source element strides */
  int64_t numel;
  uint64_t src_table;             /* const float** [ndev * n_combo]           */
  uint64_t base_off;              /* const int64_t* [ndev] (elements)          */
  uint64_t dst;                   /* float** [ndev]                            */
} spx_gather_params;

/* reduce-style (all_reduce, reduce_scatter):
 *   out[d][l] = fold_{j < n_members} src[members[d * n_members + j]] [ base_off[d] + sum_k l_k * sstride_k ] */
typedef struct {
  int32_t ndev, rank, n_members, monoid;
  int64_t dims[SPX_MAX_RANK];
  int64_t sstride[SPX_MAX_RANK];
  int64_t numel;
  uint64_t src;                   /* const float** [ndev] (device input base)  */
  uint64_t members;               /* const int32_t* [ndev * n_members]          */
  uint64_t base_off;              /* const int64_t* [ndev]                      */
  uint64_t dst;                   /* float** [ndev]                             */
  int32_t dtype, dtype_pad;
} spx_creduce_params;

/* ---- NCCL collective across processes (one mesh device per GPU) --------- */
enum spx_nccl_kind { SPX_NCCL_ALLREDUCE = 0, SPX_NCCL_ALLGATHER = 1,
                     SPX_NCCL_REDUCESCATTER = 2, SPX_NCCL_ALLTOALL = 3 };
typedef struct {
  int32_t kind, comm, monoid, pad; /* comm: index returned by spx_comm_init   */
  uint64_t send, recv;             /* device addresses                          */
  int64_t count;                   /* elements: per-rank send count (AG/A2A chunk), recv count (RS), total (AR) */
} spx_nccl_params;

/* ---- all-reduce / reduce-scatter / all-gather over NVLink peer memory ----- */
/* Flag region of a member (uint32): [slot][phase SPX_PEER_PHASES][block SPX_PEER_MAX_BLOCKS][member 8];
 * epoch counters (local): [slot][block]. */
#define SPX_PEER_MAX_BLOCKS 512
#define SPX_PEER_PHASES 3
typedef struct {
  int32_t kind, n, me, monoid;     /* kind 0 = all-reduce, 1 = all-gather (dst[m * count ..] = member m's src),
                                      2 = reduce-scatter (src[] point at my chunk of each member's input);
                                      n members; me = my index */
  int64_t count;                   /* elements (all-gather: per member) */
  uint64_t src[8];                 /* members' input buffers, mapped into this process */
  uint64_t dst;                    /* local output */
  uint64_t flags[8];               /* members' flag regions (mapped), layout above */
  uint64_t counter;                /* local epoch counters, u32 [slot][block] */
  int32_t slot, max_blocks;        /* max_blocks: 0 = default (2 per SM); fewer leave SMs to concurrent compute */
} spx_peer_params;

/* ---- host <-> device copies inside the plan ---------------------------------
 * The drop-in call's data movement as plan records: an argument's H2D copy
 * right before its first reader, a result's D2H copy right after its last
 * writer, each on its own copy stream, so the copies overlap the step instead
 * of bracketing it.  `host` must be page-locked; spx_plan_set_host rebinds it
 * before a run or a graph replay (the captured memcpy node is updated in the
 * instantiated graph). */
typedef struct {
  uint64_t dev;                    /* device address */
  uint64_t host;                   /* page-locked host address */
  uint64_t bytes;
  int32_t dir, pad;                /* 0 host->device, 1 device->host, 2 device->device: `host` is then
                                      the source device address -- possibly a peer's arena mapped
                                      by CUDA IPC (a copy-engine all-gather over NVLink) */
} spx_copy_params;

/* ---- plan records --------------------------------------------------------- */
enum spx_kind { SPX_K_EW = 1, SPX_K_REDUCE = 2, SPX_K_GEMM = 3, SPX_K_GATHER = 4,
                SPX_K_CREDUCE = 5, SPX_K_NCCL = 6, SPX_K_PEER = 7, SPX_K_SPLIT = 8, SPX_K_COPY = 9 };

/* library / device */
const char* spx_last_error(void);
int spx_version(void);
int spx_params_size(int kind);                     /* ABI check: sizeof(record params) */
int spx_device_init(int ordinal);                  /* select + check sm_100 */
int spx_malloc(uint64_t bytes, uint64_t* out_ptr);  /* arena (cudaMalloc) */
int spx_free(uint64_t ptr);
int spx_mem_info(uint64_t* free_bytes, uint64_t* total_bytes);   /* cudaMemGetInfo of the current device */
int spx_memcpy_h2d(uint64_t dst, const void* src, uint64_t bytes, uint64_t stream);
int spx_memcpy_d2h(void* dst, uint64_t src, uint64_t bytes, uint64_t stream);
int spx_memcpy_d2d(uint64_t dst, uint64_t src, uint64_t bytes, uint64_t stream);
int spx_memset(uint64_t dst, int value, uint64_t bytes, uint64_t stream);
int spx_host_alloc(uint64_t bytes, void** out_ptr); /* pinned host memory */
int spx_host_free(void* ptr);
/* page-lock / unlock an existing host range (cudaHostRegister) so copies
 * from/to it run as direct DMA at full link rate */
int spx_host_register(void* ptr, uint64_t bytes);
int spx_host_unregister(void* ptr);
/* host memcpy split over `threads` threads (staging into pinned buffers) */
int spx_host_copy(void* dst, const void* src, uint64_t bytes, int threads);
/* copies between PAGEABLE host memory and the device through a ring of pinned
 * chunks filled/drained by a host thread pool while the copy engine moves the
 * previous chunk (ordered on `stream`).  h2d returns once the source may be
 * reused; d2h returns once the data is in `dst`. */
int spx_h2d_staged(uint64_t dst, const void* src, uint64_t bytes, uint64_t stream);
int spx_d2h_staged(void* dst, uint64_t src, uint64_t bytes, uint64_t stream);
int spx_stream_create(uint64_t* out_stream);
int spx_stream_sync(uint64_t stream);
int spx_stream_destroy(uint64_t stream);

/* CUDA IPC: map another process's arena (peer collectives) */
int spx_ipc_get_handle(uint64_t ptr, uint8_t out_handle[64]);
int spx_ipc_open(const uint8_t handle[64], uint64_t* out_ptr);
int spx_ipc_close(uint64_t ptr);

/* NCCL (dlopen'd; the same libnccl torch uses) */
int spx_nccl_get_unique_id(uint8_t out_id[128]);
int spx_comm_init(const uint8_t id[128], int nranks, int rank, int* out_comm);
int spx_comm_destroy(int comm);
/* failure detection: NCCL asynchronous error of a communicator (0 = none),
 * abort, a peer-collective barrier that gave up (0 = none, else 1 + phase),
 * and a stream wait that watches for both (timeout_s 0 = no limit) */
int spx_comm_async_error(int comm, int* out_err);
int spx_comm_abort(int comm);
int spx_peer_error(int* out);
int spx_peer_error_clear(void);
int spx_stream_sync_watch(uint64_t stream, double timeout_s);

/* plans: a sequence of records [kind, param struct] executed in order on a stream */
int spx_plan_create(uint64_t* out_plan);
int spx_plan_add(uint64_t plan, int kind, const void* params, uint64_t params_bytes);
/* Scheduling (optional): run record `index` on stream `stream` (0 = the stream
 * passed to run/capture; 1..5 = the plan's side streams: 1 off-critical compute
 * such as weight-gradient GEMMs, 2 collectives (high priority), 3 parameter
 * updates, 4 host->device copies, 5 device->host copies), after the records
 * listed in `waits` (indices of earlier records on other streams) have completed.  Side streams fork from and join back into
 * the run/capture stream, so a plan stays one unit on it. */
int spx_plan_set_sched(uint64_t plan, int index, int stream, const int* waits, int n_waits);
int spx_plan_finalize(uint64_t plan);              /* builds TMA descriptors etc. */
int spx_plan_run(uint64_t plan, uint64_t stream);  /* eager launch of every record */
int spx_plan_capture(uint64_t plan, uint64_t stream);  /* record into a CUDA graph */
int spx_plan_replay(uint64_t plan, uint64_t stream);   /* launch the captured graph */
int spx_plan_launch_count(uint64_t plan);          /* kernel launches per run */
int spx_plan_destroy(uint64_t plan);
int spx_plan_record_info(uint64_t plan, int index, int* kind, int* path);

/* timing helpers (CUDA events on the given stream) */
int spx_event_create(uint64_t* out_event);
int spx_event_record(uint64_t event, uint64_t stream);
int spx_stream_wait_event(uint64_t stream, uint64_t event);   /* later work on `stream` waits */
int spx_event_elapsed_ms(uint64_t start, uint64_t end, float* out_ms);
int spx_event_destroy(uint64_t event);

/* per-record timing of one eager run (ms per record, length = record count) */
int spx_plan_profile(uint64_t plan, uint64_t stream, float* out_ms, int n);
/* Timeline of one multi-stream run (dev tool): per record, ms from the start
   of the run to the point its stream reached it with its cross-stream waits
   met (ready_ms) and to its completion (end_ms). */
int spx_plan_trace(uint64_t plan, uint64_t stream, float* ready_ms, float* end_ms, int n);

/* ---- run-time specialised elementwise kernels (csrc/ew_jit.cu) ------------
 * f32 elementwise records outside the static catalog get a kernel generated
 * from the record (program as straight-line IEEE code, shape and strides as
 * constants) and compiled by NVRTC for sm_100a when the plan is built; record
 * path -3 (spx_plan_record_info).  SPX_EW_JIT=0 keeps the interpreter.  These
 * entry points need no GPU. */
int spx_ew_jit_available(void);                 /* 1 if NVRTC loaded */
/* the generated source for a record (NUL-terminated); length or -1 */
int spx_ew_jit_source(const spx_ew_params* p, char* buf, int64_t cap);
/* generate + compile (cached by source) */
int spx_ew_jit_compile(const spx_ew_params* p);
/* the same record with the split `sp` of output `which` fused in (4-CTA
   clusters per 128 x 128 block, fp16 pieces bit-identical to the standalone
   split; skip = 1: output `which` not stored in fp32) */
int spx_ew_jit_split_source(const spx_ew_params* p, int which, int skip, char* buf, int64_t cap);
int spx_ew_jit_split_compile(const spx_ew_params* p, const spx_split_params* sp, int which, int skip);
int spx_ew_jit_stats(int* compiles, int* cached);

/* ---- executed-work accounting ---------------------------------------------
 * The reference's simulator predicts, per device, the collectives of a
 * program (`collective_counts`, spmd.py:264-271) and its FLOPs
 * (`simulate().compute_flops`, sim.py:86-100, :209-229).  The runtime counts
 * what it actually ISSUES: every eager run, profile run and graph replay adds
 * the logical collectives and FLOPs of the records it launched (a replay adds
 * what was captured into the graph).  A record's tag says which logical
 * collective it executes (one record per IR collective; relayouts around an
 * NCCL call are untagged) and whether it is internal work that the IR does
 * not contain (split-K workspace reductions: no FLOPs).  FLOPs follow the
 * simulator's convention from the record parameters: GEMM 2MNK, elementwise
 * one per arithmetic instruction per element, reduce one per input element
 * (+ the fused operand expression), summed over the record's virtual
 * devices. */
enum spx_tag_bits {
  SPX_TAG_COLL_MASK = 0x7,        /* 0 none, 1 all_gather, 2 all_reduce, 3 reduce_scatter, 4 all_to_all */
  SPX_TAG_INTERNAL = 0x100        /* no IR FLOPs (split-K partial reduction) */
};
int spx_plan_tag(uint64_t plan, int index, int tag);
int spx_plan_set_host(uint64_t plan, int index, uint64_t host);   /* SPX_K_COPY: rebind the host buffer */
typedef struct {
  int64_t runs;                   /* eager runs + graph replays + profile runs */
  int64_t coll[4];                /* logical collectives issued: all_gather, all_reduce, reduce_scatter, all_to_all */
  double flops;                   /* FLOPs issued, summed over the plan's virtual devices */
  int64_t launches;               /* kernel launches issued (graph replays count the captured launches) */
} spx_exec_stats;
int spx_plan_exec_stats(uint64_t plan, spx_exec_stats* out);
int spx_plan_reset_stats(uint64_t plan);

#ifdef __cplusplus
}
#endif
#endif
