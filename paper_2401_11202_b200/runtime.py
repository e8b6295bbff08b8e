"""ctypes binding of the C-ABI (include/spindle_b200.h).

The structures below mirror the header field for field; `check_abi()` asks
the library for its record sizes so a header/binding mismatch fails loudly.
There is no CPU fallback: if the library is missing the product path raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspindle_b200.so")

MAX_RANK, MAX_IN, MAX_OUT, MAX_PROG = 6, 8, 4, 28
NREG = 12

OP = dict(MOV=0, ADD=1, MUL=2, NEG=3, EXP=4, MAX=5, IMM=6, ADDI=7, MULI=8, IADD=9, IMUL=10)
K_EW, K_REDUCE, K_GEMM, K_GATHER, K_CREDUCE, K_NCCL = 1, 2, 3, 4, 5, 6
NCCL_ALLREDUCE, NCCL_ALLGATHER, NCCL_REDUCESCATTER, NCCL_ALLTOALL = 0, 1, 2, 3

I64R = C.c_int64 * MAX_RANK


class Insn(C.Structure):
    _fields_ = [("op", C.c_int32), ("a", C.c_int32), ("b", C.c_int32), ("dst", C.c_int32)]


class View(C.Structure):
    _fields_ = [("off", C.c_int64), ("stride", I64R)]


class EwParams(C.Structure):
    _fields_ = [("base", C.c_uint64), ("dev_stride", C.c_int64),
                ("ndev", C.c_int32), ("rank", C.c_int32), ("n_in", C.c_int32),
                ("n_out", C.c_int32), ("n_prog", C.c_int32), ("vec", C.c_int32),
                ("dtype", C.c_int32), ("dtype_pad", C.c_int32),
                ("dims", I64R), ("numel", C.c_int64),
                ("inp", View * MAX_IN),
                ("out_off", C.c_int64 * MAX_OUT), ("out_reg", C.c_int32 * MAX_OUT),
                ("prog", Insn * MAX_PROG), ("imm", C.c_float * MAX_PROG)]


class ReduceParams(C.Structure):
    _fields_ = [("x", EwParams), ("monoid", C.c_int32), ("n_kept", C.c_int32),
                ("n_red", C.c_int32), ("mode", C.c_int32),
                ("kept_dims", I64R), ("kept_stride", I64R),
                ("red_dims", I64R), ("red_stride", I64R),
                ("n_out", C.c_int64), ("n_red_elems", C.c_int64),
                ("out_off", C.c_int64), ("scratch_off", C.c_int64)]


class GemmParams(C.Structure):
    _fields_ = [("base", C.c_uint64), ("dev_stride", C.c_int64),
                ("ndev", C.c_int32), ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32),
                ("a_off", C.c_int64), ("b_off", C.c_int64), ("c_off", C.c_int64),
                ("lda", C.c_int64), ("ldb", C.c_int64), ("ldc", C.c_int64),
                ("a_mn_major", C.c_int32), ("b_k_major", C.c_int32),
                ("path", C.c_int32), ("promote", C.c_int32), ("reserve_sms", C.c_int32),
                ("splits", C.c_int32),
                ("epi", C.c_int32), ("epi_pad", C.c_int32),
                ("epi_in_off", C.c_int64 * 2), ("epi_in_ld", C.c_int64 * 2),
                ("epi_out_off", C.c_int64 * 2), ("epi_out_ld", C.c_int64 * 2),
                ("epi_imm", C.c_float * 2),
                ("sk_mode", C.c_int32), ("sk_pad", C.c_int32),
                ("ws_off", C.c_int64), ("flag_off", C.c_int64),
                ("h3_shared", C.c_int32), ("h3_splitk", C.c_int32),
                ("h3_a_off", C.c_int64), ("h3_a_scl", C.c_int64), ("h3_b_off", C.c_int64), ("h3_b_scl", C.c_int64),
                ("dtype", C.c_int32), ("dtype_pad", C.c_int32)]


class SplitParams(C.Structure):
    _fields_ = [("base", C.c_uint64), ("dev_stride", C.c_int64),
                ("ndev", C.c_int32), ("rows", C.c_int32), ("cols", C.c_int32), ("flags", C.c_int32),
                ("src_off", C.c_int64), ("ld", C.c_int64),
                ("dst_off", C.c_int64), ("pitch", C.c_int64), ("scl_off", C.c_int64)]


DT_F32, DT_I32 = 0, 1
SPLIT_PIECES_ONLY = 1
EPI_NONE, EPI_ADD, EPI_SQUARE, EPI_MULSCALE, EPI_MOMENTUM = 0, 1, 2, 3, 4


class GatherParams(C.Structure):
    _fields_ = [("ndev", C.c_int32), ("rank", C.c_int32), ("n_combo", C.c_int32), ("pad", C.c_int32),
                ("dims", I64R), ("ext", I64R), ("cmul", I64R), ("sstride", I64R),
                ("numel", C.c_int64), ("src_table", C.c_uint64), ("base_off", C.c_uint64),
                ("dst", C.c_uint64)]


class CreduceParams(C.Structure):
    _fields_ = [("ndev", C.c_int32), ("rank", C.c_int32), ("n_members", C.c_int32),
                ("monoid", C.c_int32), ("dims", I64R), ("sstride", I64R), ("numel", C.c_int64),
                ("src", C.c_uint64), ("members", C.c_uint64), ("base_off", C.c_uint64),
                ("dst", C.c_uint64), ("dtype", C.c_int32), ("dtype_pad", C.c_int32)]


class NcclParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("comm", C.c_int32), ("monoid", C.c_int32), ("pad", C.c_int32),
                ("send", C.c_uint64), ("recv", C.c_uint64), ("count", C.c_int64)]


class PeerParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("me", C.c_int32), ("monoid", C.c_int32),
                ("count", C.c_int64), ("src", C.c_uint64 * 8), ("dst", C.c_uint64),
                ("flags", C.c_uint64 * 8), ("counter", C.c_uint64), ("slot", C.c_int32),
                ("max_blocks", C.c_int32)]


K_PEER = 7
K_SPLIT = 8
K_COPY = 9


class CopyParams(C.Structure):
    _fields_ = [("dev", C.c_uint64), ("host", C.c_uint64), ("bytes", C.c_uint64), ("dir", C.c_int32),
                ("pad", C.c_int32)]

# record tags (include/spindle_b200.h spx_tag_bits)
TAG_COLL = {"all_gather": 1, "all_reduce": 2, "reduce_scatter": 3, "all_to_all": 4}
TAG_INTERNAL = 0x100
COLL_ORDER = ("all_gather", "all_reduce", "reduce_scatter", "all_to_all")


class ExecStats(C.Structure):
    _fields_ = [("runs", C.c_int64), ("coll", C.c_int64 * 4), ("flops", C.c_double), ("launches", C.c_int64)]


PEER_MAX_BLOCKS = 512      # include/spindle_b200.h
PEER_PHASES = 3

PARAMS = {K_PEER: PeerParams, K_EW: EwParams, K_REDUCE: ReduceParams, K_GEMM: GemmParams,
          K_GATHER: GatherParams, K_CREDUCE: CreduceParams, K_NCCL: NcclParams, K_SPLIT: SplitParams,
          K_COPY: CopyParams}

EXPORTS = [
    "spx_last_error", "spx_version", "spx_params_size", "spx_device_init", "spx_malloc", "spx_free",
    "spx_memcpy_h2d", "spx_memcpy_d2h", "spx_memset", "spx_stream_create", "spx_stream_sync",
    "spx_stream_destroy", "spx_nccl_get_unique_id", "spx_comm_init", "spx_comm_destroy",
    "spx_plan_create", "spx_plan_add", "spx_plan_finalize", "spx_plan_run", "spx_plan_capture",
    "spx_plan_replay", "spx_plan_launch_count", "spx_plan_destroy", "spx_plan_record_info",
    "spx_event_create", "spx_event_record", "spx_event_elapsed_ms", "spx_event_destroy",
    "spx_stream_wait_event", "spx_memcpy_d2d",
    "spx_plan_profile", "spx_plan_trace", "spx_ew_jit_available", "spx_ew_jit_source",
    "spx_ew_jit_compile", "spx_ew_jit_stats", "spx_ew_jit_split_source", "spx_ew_jit_split_compile", "spx_host_alloc", "spx_host_free", "spx_plan_set_sched",
    "spx_ipc_get_handle", "spx_ipc_open", "spx_ipc_close",
    "spx_plan_tag", "spx_plan_exec_stats", "spx_plan_reset_stats", "spx_plan_set_host",
    "spx_host_register", "spx_host_unregister", "spx_host_copy",
    "spx_h2d_staged", "spx_d2h_staged",
    "spx_mem_info", "spx_h3_range_events",
    "spx_comm_async_error", "spx_comm_abort", "spx_peer_error", "spx_peer_error_clear", "spx_stream_sync_watch",
]

_lib = None


class BackendError(RuntimeError):
    pass


def load(build_if_missing: bool = True):
    """Load libspindle_b200.so (building it in-tree if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from .build import build
        build()
    if not os.path.exists(LIB_PATH):
        raise BackendError(f"{LIB_PATH} missing: the CUDA backend is not built "
                           "(python -m paper_2401_11202_b200.build)")
    lib = C.CDLL(LIB_PATH)
    lib.spx_last_error.restype = C.c_char_p
    u64p = C.POINTER(C.c_uint64)
    sigs = {
        "spx_malloc": [C.c_uint64, u64p], "spx_free": [C.c_uint64],
        "spx_memcpy_h2d": [C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64],
        "spx_memcpy_d2h": [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64],
        "spx_memset": [C.c_uint64, C.c_int, C.c_uint64, C.c_uint64],
        "spx_stream_create": [u64p], "spx_stream_sync": [C.c_uint64],
        "spx_stream_destroy": [C.c_uint64],
        "spx_plan_create": [u64p], "spx_plan_add": [C.c_uint64, C.c_int, C.c_void_p, C.c_uint64],
        "spx_plan_finalize": [C.c_uint64], "spx_plan_run": [C.c_uint64, C.c_uint64],
        "spx_plan_capture": [C.c_uint64, C.c_uint64], "spx_plan_replay": [C.c_uint64, C.c_uint64],
        "spx_plan_launch_count": [C.c_uint64], "spx_plan_destroy": [C.c_uint64],
        "spx_plan_record_info": [C.c_uint64, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "spx_event_create": [u64p], "spx_event_record": [C.c_uint64, C.c_uint64],
        "spx_stream_wait_event": [C.c_uint64, C.c_uint64],
        "spx_memcpy_d2d": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64],
        "spx_event_elapsed_ms": [C.c_uint64, C.c_uint64, C.POINTER(C.c_float)],
        "spx_event_destroy": [C.c_uint64],
        "spx_plan_profile": [C.c_uint64, C.c_uint64, C.POINTER(C.c_float), C.c_int],
        "spx_plan_trace": [C.c_uint64, C.c_uint64, C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int],
        "spx_ew_jit_available": [],
        "spx_ew_jit_source": [C.c_void_p, C.c_char_p, C.c_int64],
        "spx_ew_jit_compile": [C.c_void_p],
        "spx_ew_jit_stats": [C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "spx_ew_jit_split_source": [C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_int64],
        "spx_ew_jit_split_compile": [C.c_void_p, C.c_void_p, C.c_int, C.c_int],
        "spx_nccl_get_unique_id": [C.c_void_p],
        "spx_comm_init": [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int)],
        "spx_comm_destroy": [C.c_int], "spx_device_init": [C.c_int], "spx_params_size": [C.c_int],
        "spx_host_alloc": [C.c_uint64, C.POINTER(C.c_void_p)], "spx_host_free": [C.c_void_p],
        "spx_plan_set_sched": [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int],
        "spx_ipc_get_handle": [C.c_uint64, C.c_void_p], "spx_ipc_open": [C.c_void_p, C.POINTER(C.c_uint64)],
        "spx_ipc_close": [C.c_uint64],
        "spx_plan_tag": [C.c_uint64, C.c_int, C.c_int],
        "spx_plan_set_host": [C.c_uint64, C.c_int, C.c_uint64],
        "spx_mem_info": [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
        "spx_h3_range_events": [C.POINTER(C.c_uint32), C.c_int],
        "spx_plan_exec_stats": [C.c_uint64, C.POINTER(ExecStats)],
        "spx_plan_reset_stats": [C.c_uint64],
        "spx_host_register": [C.c_void_p, C.c_uint64], "spx_host_unregister": [C.c_void_p],
        "spx_host_copy": [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int],
        "spx_h2d_staged": [C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64],
        "spx_d2h_staged": [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64],
        "spx_comm_async_error": [C.c_int, C.POINTER(C.c_int)], "spx_comm_abort": [C.c_int],
        "spx_peer_error": [C.POINTER(C.c_int)], "spx_peer_error_clear": [],
        "spx_stream_sync_watch": [C.c_uint64, C.c_double],
    }
    for name, args in sigs.items():
        getattr(lib, name).argtypes = args
    _lib = lib
    check_abi(lib)
    return lib


def check_abi(lib):
    for kind, cls in PARAMS.items():
        n = lib.spx_params_size(kind)
        if n != C.sizeof(cls):
            raise BackendError(f"ABI mismatch for record kind {kind}: C {n} bytes, Python {C.sizeof(cls)}")


def call(fn, *args):
    rc = fn(*args)
    if rc != 0:
        raise BackendError(_lib.spx_last_error().decode(errors="replace"))
    return rc


class Device:
    """One GPU: arena allocations + a stream."""

    def __init__(self, ordinal: int = 0):
        self.lib = load()
        self.ordinal = ordinal
        call(self.lib.spx_device_init, ordinal)
        s = C.c_uint64()
        call(self.lib.spx_stream_create, C.byref(s))
        self.stream = s.value
        self._allocs = []
        self._pinned = []

    def malloc(self, nbytes: int) -> int:
        p = C.c_uint64()
        call(self.lib.spx_malloc, int(nbytes), C.byref(p))
        self._allocs.append(p.value)
        return p.value

    def mem_info(self) -> tuple[int, int]:
        """(free, total) device bytes."""
        f, t = C.c_uint64(), C.c_uint64()
        call(self.lib.spx_mem_info, C.byref(f), C.byref(t))
        return f.value, t.value

    def free(self, ptr: int):
        if ptr in self._allocs:
            self._allocs.remove(ptr)
            call(self.lib.spx_free, ptr)

    def h2d(self, dst: int, arr: np.ndarray):
        arr = np.ascontiguousarray(arr)
        call(self.lib.spx_memcpy_h2d, dst, arr.ctypes.data, arr.nbytes, self.stream)

    def d2h(self, arr: np.ndarray, src: int):
        assert arr.flags.c_contiguous
        call(self.lib.spx_memcpy_d2h, arr.ctypes.data, src, arr.nbytes, self.stream)

    def h2d_staged(self, dst: int, arr: np.ndarray):
        """Pageable host array -> device through pinned staging (spx_h2d_staged)."""
        arr = np.ascontiguousarray(arr)
        call(self.lib.spx_h2d_staged, dst, arr.ctypes.data, arr.nbytes, self.stream)

    def d2h_staged(self, arr: np.ndarray, src: int):
        """Device -> pageable host array through pinned staging; returns when
        `arr` holds the data (spx_d2h_staged)."""
        assert arr.flags.c_contiguous
        call(self.lib.spx_d2h_staged, arr.ctypes.data, src, arr.nbytes, self.stream)

    def memset(self, dst: int, nbytes: int, value: int = 0):
        call(self.lib.spx_memset, dst, value, nbytes, self.stream)

    def sync(self):
        call(self.lib.spx_stream_sync, self.stream)

    def sync_watch(self, timeout_s: float | None = None):
        """Wait for the stream while watching for NCCL asynchronous errors and
        peer-collective timeouts (spx_stream_sync_watch); raises BackendError."""
        if timeout_s is None:
            timeout_s = float(os.environ.get("SPX_SYNC_TIMEOUT_S", "900"))
        call(self.lib.spx_stream_sync_watch, self.stream, timeout_s)

    def event(self) -> int:
        e = C.c_uint64()
        call(self.lib.spx_event_create, C.byref(e))
        return e.value

    def record(self, ev: int, stream: int | None = None):
        call(self.lib.spx_event_record, ev, self.stream if stream is None else stream)

    def new_stream(self) -> int:
        s = C.c_uint64()
        call(self.lib.spx_stream_create, C.byref(s))
        return s.value

    def wait(self, ev: int, stream: int | None = None):
        """Work issued later on `stream` (default: the device stream) waits for `ev`."""
        call(self.lib.spx_stream_wait_event, self.stream if stream is None else stream, ev)

    def h2d_async(self, dst: int, arr: np.ndarray, stream: int):
        call(self.lib.spx_memcpy_h2d, dst, arr.ctypes.data, arr.nbytes, stream)

    def d2d(self, dst: int, src: int, nbytes: int, stream: int | None = None):
        call(self.lib.spx_memcpy_d2d, dst, src, nbytes, self.stream if stream is None else stream)

    def elapsed_ms(self, a: int, b: int) -> float:
        out = C.c_float()
        call(self.lib.spx_event_elapsed_ms, a, b, C.byref(out))
        return float(out.value)

    def pinned(self, shape, dtype=np.float32) -> np.ndarray:
        """Pinned (page-locked) host array for async H2D/D2H."""
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        call(self.lib.spx_host_alloc, max(nbytes, 16), C.byref(p))
        buf = (C.c_uint8 * max(nbytes, 16)).from_address(p.value)
        arr = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype).reshape(shape)
        self._pinned.append(p.value)
        return arr

    def close(self):
        for p in list(self._allocs):
            self.free(p)
        for p in self._pinned:
            self.lib.spx_host_free(C.c_void_p(p))
        self._pinned = []


def h3_range_events(reset: bool = True) -> int:
    """Operand blocks whose fp16-split scale was clamped since the last reset
    (include/spindle_b200.h spx_h3_range_events)."""
    out = C.c_uint32()
    call(load().spx_h3_range_events, C.byref(out), 1 if reset else 0)
    return int(out.value)


class PinnedPool:
    """Page-locked host arrays for the drop-in call's results.

    `array()` hands out a NEW numpy array (owned by the caller) backed by a
    pinned buffer; when the caller drops the last reference the buffer goes
    back to the pool (weakref finalizer) and serves a later result of the same
    size.  Results then come back by direct DMA (~57 GB/s on this box) instead
    of pageable copies into freshly faulted pages (~5 GB/s), and a result fed
    back as the next call's input -- a training loop's parameters and momenta
    -- goes in by direct DMA too (`contains`).  Bounded by
    SPX_PINNED_POOL_BYTES (default 64 GiB); beyond it callers get ordinary
    arrays.  SPX_PINNED_POOL=0 disables it."""

    def __init__(self, lib):
        import threading
        self.lib = lib
        self.limit = int(os.environ.get("SPX_PINNED_POOL_BYTES", str(64 << 30)))
        self.enabled = os.environ.get("SPX_PINNED_POOL", "1") != "0"
        self.free: dict[int, list[int]] = {}
        self.ranges: dict[int, int] = {}       # ptr -> nbytes of every pinned buffer
        self._starts: list[int] = []
        self.total = 0
        self.lock = threading.Lock()

    def _release(self, ptr: int, nbytes: int):
        with self.lock:
            self.free.setdefault(nbytes, []).append(ptr)

    def array(self, shape, dtype) -> np.ndarray | None:
        dtype = np.dtype(dtype)
        nbytes = max(16, int(np.prod(shape)) * dtype.itemsize)
        if not self.enabled:
            return None
        with self.lock:
            lst = self.free.get(nbytes)
            ptr = lst.pop() if lst else None
            if ptr is None:
                if self.total + nbytes > self.limit:
                    return None
                p = C.c_void_p()
                call(self.lib.spx_host_alloc, nbytes, C.byref(p))
                ptr = p.value
                self.total += nbytes
                self.ranges[ptr] = nbytes
                import bisect
                bisect.insort(self._starts, ptr)
        import weakref
        buf = (C.c_uint8 * nbytes).from_address(ptr)
        weakref.finalize(buf, self._release, ptr, nbytes)
        n = int(np.prod(shape))
        return np.frombuffer(buf, dtype=dtype, count=n).reshape(shape)

    def contains(self, arr: np.ndarray) -> bool:
        """Is `arr` (contiguous) inside a pinned buffer of this pool?"""
        if not self._starts:
            return False
        import bisect
        a = arr.ctypes.data
        i = bisect.bisect_right(self._starts, a) - 1
        if i < 0:
            return False
        s = self._starts[i]
        return a + arr.nbytes <= s + self.ranges[s]


_POOL = None


def pinned_pool() -> PinnedPool:
    global _POOL
    if _POOL is None:
        _POOL = PinnedPool(load())
    return _POOL


class NativePlan:
    """A finalized sequence of records on one device."""

    def __init__(self, device: Device):
        self.dev = device
        self.lib = device.lib
        h = C.c_uint64()
        call(self.lib.spx_plan_create, C.byref(h))
        self.h = h.value
        self.n_records = 0
        self.captured = False

    def add(self, kind: int, params):
        assert isinstance(params, PARAMS[kind])
        call(self.lib.spx_plan_add, self.h, kind, C.byref(params), C.sizeof(params))
        self.n_records += 1

    def tag(self, index: int, tag: int):
        call(self.lib.spx_plan_tag, self.h, index, tag)

    def set_host(self, index: int, host: int):
        """Rebind a copy record's page-locked host buffer (also in the captured graph)."""
        call(self.lib.spx_plan_set_host, self.h, index, host)

    def exec_stats(self) -> dict:
        """What the runtime has issued so far (include/spindle_b200.h spx_exec_stats)."""
        st = ExecStats()
        call(self.lib.spx_plan_exec_stats, self.h, C.byref(st))
        return {"runs": int(st.runs), "coll": {k: int(st.coll[i]) for i, k in enumerate(COLL_ORDER)},
                "flops": float(st.flops), "launches": int(st.launches)}

    def reset_stats(self):
        call(self.lib.spx_plan_reset_stats, self.h)

    def set_sched(self, index: int, stream: int, waits):
        arr = (C.c_int * max(1, len(waits)))(*waits)
        call(self.lib.spx_plan_set_sched, self.h, index, stream, arr, len(waits))

    def finalize(self):
        call(self.lib.spx_plan_finalize, self.h)

    def run(self):
        call(self.lib.spx_plan_run, self.h, self.dev.stream)

    def capture(self):
        call(self.lib.spx_plan_capture, self.h, self.dev.stream)
        self.captured = True

    def replay(self):
        call(self.lib.spx_plan_replay, self.h, self.dev.stream)

    def launch_count(self) -> int:
        return int(self.lib.spx_plan_launch_count(self.h))

    def record_info(self, i: int):
        k, p = C.c_int(), C.c_int()
        call(self.lib.spx_plan_record_info, self.h, i, C.byref(k), C.byref(p))
        return k.value, p.value

    def profile(self) -> np.ndarray:
        out = (C.c_float * self.n_records)()
        call(self.lib.spx_plan_profile, self.h, self.dev.stream, out, self.n_records)
        return np.array(out[:], dtype=np.float64)

    def trace(self) -> tuple:
        """One multi-stream run with per-record (ready, end) times in ms."""
        r = (C.c_float * self.n_records)()
        e = (C.c_float * self.n_records)()
        call(self.lib.spx_plan_trace, self.h, self.dev.stream, r, e, self.n_records)
        return np.array(r[:], dtype=np.float64), np.array(e[:], dtype=np.float64)

    def destroy(self):
        if self.h:
            self.lib.spx_plan_destroy(self.h)
            self.h = 0

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
