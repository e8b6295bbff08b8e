"""Executable: arena layout + native plan for one compiled localized function.

Two hosting modes for the mesh devices of a localized module:

  "local"  every mesh device lives on this process's GPU (virtual devices at
           a fixed arena stride); collectives are in-GPU group kernels --
           this is the drop-in `spmd_interpret` mode and what the parity tests
           exercise on a single B200;
  "nccl"   one process per GPU and mesh device (torchrun); collectives are
           NCCL calls on per-group communicators, with in-GPU relayouts where
           the chunk order of a layout differs from the communicator order.

Layout of one device slice of the arena: [args | liveness-packed
intermediates and results | reduce scratch], identical on every device.
"""
from __future__ import annotations

import ctypes as C
import os as _os

import numpy as np

from . import runtime as R
from .plan import ALIGN, Compiler, Kernel, Leaf, Node, Program, UnsupportedProgram, _align, _contig, _prod


def _collapse(dims, views):
    """Merge adjacent dims where every view is mergeable (contiguous or both 0)."""
    dims = list(dims)
    views = [list(v) for v in views]
    k = len(dims) - 2
    while k >= 0:
        ok = all(v[k] == v[k + 1] * dims[k + 1] for v in views)
        if ok:
            dims[k] = dims[k] * dims[k + 1]
            del dims[k + 1]
            for v in views:
                v[k] = v[k + 1]
                del v[k + 1]
        k -= 1
    return dims, views


class Executable:
    DRY_BASE = 1 << 40
    DRY_TABLES = 1 << 44

    def __init__(self, module, func="main", device: R.Device | None = None, devices=None,
                 comm_mode="local", comms=None, gemm_path=0, dry=False, comm_factory=None,
                 overlap=None, dtype=np.float32, io=False, before_alloc=None):
        """dry=True builds the records against fake addresses without a GPU
        (used by the CPU tests and the record simulator).  dtype: the
        arithmetic type of the call (np.result_type of the inputs,
        evaluator._cdtype): float32 or int32.  io=True: the plan also copies
        its arguments in and its results out (SPX_K_COPY records on two copy
        streams, each right next to its first reader / last writer) -- the
        drop-in call's data movement overlapped with the step (`call`)."""
        self.dtype = np.dtype(dtype)
        self.dt = R.DT_I32 if self.dtype == np.dtype(np.int32) else R.DT_F32
        if self.dt == R.DT_I32 and comm_mode != "local":
            raise TypeError("int32 programs run in local mode (the drop-in spmd_interpret / interpret)")
        h3 = gemm_path == 0 and _os.environ.get("SPX_GEMM_H3", "1") != "0" and self.dtype == np.float32
        self.comp = Compiler(module, func, devices=devices, comm_mode=comm_mode, dtype=self.dtype, h3=h3).compile()
        self.dry = dry
        self.device = None if dry else (device or R.Device(0))
        self.ndev = len(self.comp.devices)
        self.mesh_size = module.mesh.device_count if getattr(module, "mesh", None) is not None else 1
        self.gemm_path = gemm_path
        self.comms = comms or {}
        self._own_comms = False
        import os
        if overlap is None:
            overlap = os.environ.get("SPX_OVERLAP", "1") != "0"
        if overlap:
            self._hoist_terminal()
        self._share_splits()
        self.io = io
        if io:
            self._add_copies()
        self.stream_of = self._streams() if overlap else {}
        self.side = set(self.stream_of)
        self.overlap = bool(self.side)
        self.reserve_sms = int(os.environ.get("SPX_RESERVE_SMS", "0")) if self.overlap else 0
        # NCCL mode: critical-path all-reduces as one-shot NVLink peer-memory
        # reductions (csrc/peer.cu) once the factory maps the peers' arenas
        self.wants_peer = comm_mode == "nccl" and os.environ.get("SPX_PEER", "1") != "0"
        self.peer_max_bytes = int(os.environ.get("SPX_PEER_MAX_BYTES", str(64 << 20)))
        self.peer_ag = os.environ.get("SPX_PEER_AG", "1") != "0"
        self.peer_ag_all = os.environ.get("SPX_PEER_AG_ALL", "1") != "0"
        self.peer_rs = os.environ.get("SPX_PEER_RS", "1") != "0"
        self.peer_side_blocks = int(os.environ.get("SPX_PEER_SIDE_BLOCKS", "0"))
        # large off-critical peer collectives (C3's 64 MB gradient reduce-scatters,
        # now overlapped with the backward GEMMs since they are hoisted) run on
        # 32 blocks so the GEMMs keep the other SMs: C3 N=4 129.2k -> 137.2k;
        # smaller ones (C2/C5 gradient all-reduces, <= 16 MB) keep the full grid
        # (profiles/r02_hoist_variants_n4.txt)
        self.peer_offcrit_blocks = int(os.environ.get("SPX_PEER_OFFCRIT_BLOCKS", "32"))
        self.peer_offcrit_min_bytes = int(os.environ.get("SPX_PEER_OFFCRIT_MIN_BYTES", str(32 << 20)))
        self.ce_ag = os.environ.get("SPX_CE_AG", "1") != "0"
        self.ce_rs = os.environ.get("SPX_CE_RS", "0") != "0"
        self.peer_prebarrier = os.environ.get("SPX_PEER_PREBARRIER", "0") != "0"
        # copy-engine collectives pay a DMA setup per copy (~5-10 us): only large
        # ones gain (C3's 16-64 MB parameter gathers +2.6%, C5's 4-8 MB ones -17%
        # at N=4, profiles/r02_ce_ag_n4.txt)
        self.ce_min_bytes = int(os.environ.get("SPX_CE_MIN_BYTES", str(16 << 20)))
        self.one_stream = comm_mode == "nccl" and os.environ.get("SPX_COLL_ONE_STREAM", "1") != "0"
        self.peer_bases = None          # [arena base of rank r, mapped here]
        self._peer_handles = []
        self._layout()
        if before_alloc is not None and not dry:
            before_alloc(self.slice_elems * 4 * self.ndev)    # e.g. the plan cache evicting to make room
        self._alloc()
        if comm_mode == "nccl" and comm_factory is not None:
            self.comms = comm_factory(self)
            self._own_comms = not dry
        self._tables = []
        self._records = []
        self._krange = []          # per compiler kernel: [first record, end record)
        self.copy_in, self.copy_out = {}, {}   # (arg, device) / (result j, device) -> copy record

        self._emit()
        self._upload_tables()
        # collectives on a side stream, overlapped with compute (NCCL mode)
        self.sched = self._schedule() if self.overlap else []
        self.plan = None
        if not dry:
            self.plan = R.NativePlan(self.device)
            for kind, params in self._records:
                self.plan.add(kind, params)
            for idx, tag in self._tags.items():
                self.plan.tag(idx, tag)
            for idx, stream, waits in self.sched:
                self.plan.set_sched(idx, stream, waits)
            self.plan.finalize()

    # ---------------------------------------------------------------- layout
    def _layout(self):
        c = self.comp
        ks = c.kernels
        n = len(ks)
        first, last = {}, {}
        for i, k in enumerate(ks):
            for b in k.outs:
                first.setdefault(b, i)
            for b in k.ins:
                last[b] = max(last.get(b, -1), i)
            # a split right after the elementwise kernel that produces its
            # source may run INSIDE that kernel (runtime.cu: ew_static_split):
            # its pieces must not reuse the producer's inputs, which other
            # CTAs of the fused launch may still be reading
            if k.kind == "split" and i > 0 and ks[i - 1].kind == "ew" and k.data["src"][0] in ks[i - 1].outs:
                for b in ks[i - 1].ins:
                    last[b] = max(last.get(b, -1), i)
        off = {}
        top = 0
        for a in c.arg_bufs:
            off[a] = top
            top += _align(c.buffers[a])
        base = top
        keep = set(c.result_bufs)
        if self.overlap:
            # buffers a side-stream kernel touches are not recycled: reuse would
            # add write-after-read edges that serialise the two streams
            for i, k in enumerate(ks):
                if i in self.side:
                    keep.update(k.ins)
                    keep.update(k.outs)
        free: list[tuple[int, int]] = []   # (offset, size) holes above `base`
        hi = base
        order = sorted((first[b], b) for b in first if b not in off)
        by_start: dict[int, list[str]] = {}
        for i, b in order:
            by_start.setdefault(i, []).append(b)
        by_end: dict[int, list[str]] = {}
        for b, e in last.items():
            if b in off and b in c.arg_bufs:
                continue
            by_end.setdefault(e, []).append(b)

        def alloc(size):
            nonlocal hi
            for j, (o, s) in enumerate(free):
                if s >= size:
                    if s == size:
                        free.pop(j)
                    else:
                        free[j] = (o + size, s - size)
                    return o
            o = hi
            hi += size
            return o

        def release(o, size):
            free.append((o, size))
            free.sort()
            merged = []
            for fo, fs in free:
                if merged and merged[-1][0] + merged[-1][1] == fo:
                    merged[-1] = (merged[-1][0], merged[-1][1] + fs)
                else:
                    merged.append((fo, fs))
            free[:] = merged

        for i in range(n):
            for b in by_start.get(i, []):
                off[b] = alloc(_align(c.buffers[b]))
            for b in by_end.get(i, []):
                if b in keep or b not in off or b in c.arg_bufs:
                    continue
                if first.get(b, -1) > i:
                    continue
                release(off[b], _align(c.buffers[b]))
            for b in ks[i].outs:          # written but never read and not returned
                if b not in last and b not in keep:
                    release(off[b], _align(c.buffers[b]))
        scratch = 0
        for k in ks:
            if k.kind == "reduce":
                n_out = _prod(d for j, d in enumerate(k.data["in_dims"]) if j not in k.data["red"])
                scratch = max(scratch, 20480 + 2 * n_out)
        self.scratch_off = hi
        hi += _align(scratch)
        # zero page: source for all_gather chunks no device owns (a layout that
        # repeats an axis, e.g. [["M", "M"]], leaves zero-filled chunks exactly
        # like the reference's np.zeros buffer, spmd_interp.py:86)
        zero = 0
        for k in ks:
            if k.kind == "coll" and k.data["kind"] == "all_gather":
                zero = max(zero, _prod(k.data["in_dims"]))
        self.zero_off = hi
        self.zero_elems = _align(zero) if zero else 0
        hi += self.zero_elems
        # NCCL mode: staging for collectives whose chunk order differs from the
        # communicator's rank order (send/recv relayouts around the NCCL call)
        stage = 0
        if c.comm_mode == "nccl":
            for k in ks:
                if k.kind == "coll" and k.data["kind"] != "all_slice":
                    stage = max(stage, _prod(k.data["in_dims"]), _prod(k.data["out_dims"]))
        self.stage_elems = _align(stage)
        self.stage_a = hi
        self.stage_b = hi + self.stage_elems
        hi += 2 * self.stage_elems
        # peer collectives: flag words [comm key][phase][member] (written by the
        # peers through their mapping of this arena) and local epoch counters
        nkeys = len(self.peer_slots()) if c.comm_mode == "nccl" else 0
        self.n_peer_slots = nkeys
        self.flag_off = hi
        self.counter_off = hi + nkeys * R.PEER_PHASES * R.PEER_MAX_BLOCKS * 8
        self.flag_elems = (_align(nkeys * R.PEER_PHASES * R.PEER_MAX_BLOCKS * 8 + nkeys * R.PEER_MAX_BLOCKS)
                           if nkeys else 0)
        hi += self.flag_elems
        # in-kernel split-K (critical-path GEMMs, serialised on the main
        # stream): one shared partial workspace and one flag array (uint32,
        # zero between launches)
        ws = fl = 0
        for k in ks:
            if k.kind == "gemm" and k.data.get("sk_inkernel"):
                d = k.data
                ws = max(ws, (d["splits"] - 1) * d["M"] * d["N"])
                fl = max(fl, -(-d["M"] // 256) * -(-d["N"] // 128) * 2 * 4)
        self.sk_ws_off = hi
        hi += _align(ws) if ws else 0
        self.sk_flag_off = hi
        self.sk_flag_elems = _align(fl) if fl else 0
        hi += self.sk_flag_elems
        self.off = off
        self.slice_elems = _align(hi, 1 << 18)           # 1 MiB granularity per device
        self.peak_bytes = hi * 4

    def _alloc(self):
        self.dev_stride = self.slice_elems * 4
        self.base = self.DRY_BASE if self.dry else self.device.malloc(self.dev_stride * self.ndev)
        if self.zero_elems and not self.dry:
            self.device.memset(self.base + self.zero_off * 4, self.zero_elems * 4, 0)
        if self.flag_elems and not self.dry:
            self.device.memset(self.base + self.flag_off * 4, self.flag_elems * 4, 0)
        if self.sk_flag_elems and not self.dry:
            for p in range(self.ndev):
                self.device.memset(self.base + p * self.dev_stride + self.sk_flag_off * 4, self.sk_flag_elems * 4, 0)

    def addr(self, p: int, buf: str, extra: int = 0) -> int:
        return self.base + p * self.dev_stride + (self.off[buf] + extra) * 4

    # ---------------------------------------------------------------- tables
    def _table(self, arr: np.ndarray) -> int:
        """Queue a device table; returns a placeholder index resolved at upload."""
        self._tables.append(np.ascontiguousarray(arr))
        return len(self._tables) - 1

    def _upload_tables(self):
        sizes = [_align(t.nbytes, 16) for t in self._tables]
        total = max(16, sum(sizes))
        self.table_base = self.DRY_TABLES if self.dry else self.device.malloc(total)
        blob = np.zeros(total, dtype=np.uint8)
        addrs, o = [], 0
        for t, s in zip(self._tables, sizes):
            blob[o:o + t.nbytes] = t.view(np.uint8).reshape(-1)
            addrs.append(self.table_base + o)
            o += s
        self.table_blob = blob
        if not self.dry:
            self.device.h2d(self.table_base, blob)
            self.device.sync()
        for kind, p in self._records:
            for fld in ("src_table", "base_off", "dst", "src", "members"):
                if hasattr(p, fld) and isinstance(getattr(p, fld), int) and getattr(p, fld) >= (1 << 62):
                    setattr(p, fld, addrs[getattr(p, fld) - (1 << 62)])

    def _tref(self, arr) -> int:
        return (1 << 62) + self._table(arr)

    # ------------------------------------------------------------------ emit
    def _ew_params(self, exprs: dict, dims, outs_keep=None) -> R.EwParams:
        prog = Program.build(exprs)
        names = list(exprs)
        dims = tuple(dims) if dims else (1,)
        views = [list(l.strides) if len(l.strides) else [1] for l in prog.leaves]
        views = [v if len(v) == len(dims) else [0] * len(dims) for v in views]
        cdims, cviews = _collapse(dims, [v for v in views] + [list(_contig(dims))])
        cviews = cviews[:-1]
        p = R.EwParams()
        p.base = self.base
        p.dev_stride = self.dev_stride
        p.ndev = self.ndev
        p.rank = len(cdims)
        p.n_in = len(prog.leaves)
        p.numel = _prod(dims)
        for k, d in enumerate(cdims):
            p.dims[k] = d
        vec = 1 if (p.numel % 4 == 0 and cdims[-1] % 4 == 0) else 0
        for j, (l, v) in enumerate(zip(prog.leaves, cviews)):
            p.inp[j].off = self.off[l.buf] + l.off
            for k, s in enumerate(v):
                p.inp[j].stride[k] = s
            if v[-1] not in (0, 1):
                vec = 0
            if v[-1] == 1 and (p.inp[j].off % 4 or any(s % 4 for s in v[:-1])):
                vec = 0
        keep = outs_keep or names
        p.n_out = len(keep)
        for o, name in enumerate(keep):
            p.out_off[o] = self.off[name]
            p.out_reg[o] = prog.out_regs[names.index(name)]
        p.n_prog = len(prog.insns)
        for i, (op, a, b, dst, imm) in enumerate(prog.insns):
            p.prog[i].op, p.prog[i].a, p.prog[i].b, p.prog[i].dst = op, a, b, dst
            p.imm[i] = self._imm(imm)
        p.vec = vec
        p.dtype = self.dt
        return p

    def _imm(self, v) -> float:
        """Immediate as stored in the record: the f32 value, or the int32 bits
        (SPX_DT_I32 records reinterpret imm[])."""
        if self.dt == R.DT_I32:
            return float(np.array([v], dtype=np.int32).view(np.float32)[0])
        return float(v)

    def _emit(self):
        c = self.comp
        self._tags = {}
        for i, k in enumerate(c.kernels):
            first = len(self._records)
            self._cur = i
            self._emit_one(k)
            end = len(self._records)
            self._krange.append((first, end))
            # the record that executes the logical collective (local mode: the
            # group kernel; NCCL mode: the NCCL call or peer kernel, not the
            # relayouts around it) and internal work without IR FLOPs
            if k.kind == "coll" and k.data["kind"] in R.TAG_COLL and end > first:
                idx = next((r for r in range(first, end) if self._records[r][0] in (R.K_NCCL, R.K_PEER)),
                           next((r for r in range(first, end) if self._records[r][0] == R.K_COPY), first))
                self._tags[idx] = R.TAG_COLL[k.data["kind"]]
            if k.data.get("internal"):
                for r in range(first, end):
                    self._tags[r] = self._tags.get(r, 0) | R.TAG_INTERNAL

    def _emit_one(self, k):
        c = self.comp
        if True:
            if k.kind == "ew":
                self._records.append((R.K_EW, self._ew_params(k.data["exprs"], k.data["dims"],
                                                              k.data.get("outs_keep"))))
            elif k.kind == "reduce":
                self._emit_reduce(k)
            elif k.kind == "gemm":
                self._emit_gemm(k)
            elif k.kind == "split":
                self._emit_split(k)
            elif k.kind == "copy":
                self._emit_copy(k)
            elif k.kind == "coll":
                if c.comm_mode == "local":
                    self._emit_coll_local(k)
                else:
                    self._emit_coll_nccl(k)

    def _h3_eligible(self, d) -> bool:
        """The block-scaled 3xFP16 kernel takes this GEMM (runtime.cu h3_default,
        gemm_h3.cu spx_gemm_h3_supported, gemm_tc.cu spx_gemm_tc_supported)."""
        import os
        if self.gemm_path != 0 or os.environ.get("SPX_GEMM_H3", "1") == "0" or self.dt != R.DT_F32:
            return False
        if d.get("splits", 1) != 1 or d.get("epi") is not None or d.get("sk_inkernel") or not d.get("tc_ok"):
            return False
        (_, aoff, lda, _), (_, boff, ldb, _) = d["a"], d["b"]
        return (aoff % 4 == 0 and boff % 4 == 0 and lda % 4 == 0 and ldb % 4 == 0
                and d["M"] >= 64 and d["N"] >= 32 and d["K"] >= 32)

    def _share_splits(self):
        """One SPX_K_SPLIT per distinct fp32 operand view of the 3xFP16 GEMMs.
        Buffers are single-assignment, so the fp16 pieces of a tensor serve
        every GEMM that reads the same view -- a weight in the forward GEMM and,
        transposed, in the input-gradient GEMM; an activation in the forward
        GEMM and in the weight-gradient GEMM (128 x 128 scale blocks are
        symmetric, the GEMM reads either orientation).  The split kernel runs
        just before the first GEMM that needs it."""
        import os
        if os.environ.get("SPX_H3_SHARE", "1") == "0":
            return
        c = self.comp
        out = []
        made = {}
        args = set(c.arg_bufs)
        pre = []            # splits of function arguments (weights, the batch): no producer, hoisted
        producer = {}
        for k in c.kernels:
            for b in k.outs:
                producer[b] = k
        after: dict = {}    # elementwise producer -> splits of its outputs (fused into it by the runtime)
        self.n_splits = 0
        for k in c.kernels:
            if k.kind == "gemm" and self._h3_eligible(k.data):
                d = k.data
                M, N, K = d["M"], d["N"], d["K"]
                for side, (buf, off, ld, t), shape in (("a", d["a"], (K, M) if d["a"][3] else (M, K)),
                                                       ("b", d["b"], (N, K) if d["b"][3] else (K, N))):
                    rows, cols = shape
                    key = (buf, off, ld, rows, cols)
                    if key not in made:
                        pitch = (cols + 7) // 8 * 8
                        pieces = _align(rows * pitch)          # [2][rows][pitch] halves = rows * pitch floats
                        scl = -(-rows // 128) * -(-cols // 128)
                        name = f"%h3#{len(made)}"
                        c.buffers[name] = pieces + scl
                        c.bufdims[name] = (pieces + scl,)
                        made[key] = name
                        sk = Kernel("split", [name], {buf}, op_index=k.op_index,
                                    data=dict(src=(buf, off, ld), rows=rows, cols=cols, pitch=pitch,
                                              scl_off=pieces))
                        pk = producer.get(buf)
                        if buf in args and os.environ.get("SPX_SPLIT_PREFETCH", "1") != "0":
                            pre.append(sk)
                        elif pk is not None and pk.kind == "ew" and off == 0 and ld == cols:
                            after.setdefault(id(pk), []).append(sk)
                            sk.data["fusable"] = True
                        else:
                            out.append(sk)
                        self.n_splits += 1
                    k.ins = set(k.ins) | {made[key]}
                    d["h3" + side] = made[key]
                    d["h3" + side + "_scl"] = c.bufdims[made[key]][0] - (-(-rows // 128) * -(-cols // 128))
            out.append(k)
        final = list(pre)
        for k in out:
            final.append(k)
            final.extend(after.get(id(k), []))
        c.kernels = final
        # A fused split's source that every reader takes through its pieces (h3
        # GEMMs reading this very split) and that is no result need not be stored
        # in fp32 by the producing launch (SPX_SPLIT_PIECES_ONLY; the runtime
        # honours it only when it really fuses the split into that launch).
        results = set(c.result_bufs)
        for k in final:
            if k.kind != "split" or not k.data.get("fusable"):
                continue
            src = k.data["src"][0]
            name = k.outs[0]
            ok = src not in results
            for r in final:
                if r is k or src not in r.ins:
                    continue
                if not (r.kind == "gemm" and name in (r.data.get("h3a"), r.data.get("h3b"))):
                    ok = False
                    break
                (ab, _, _, _), (bb, _, _, _) = r.data["a"], r.data["b"]
                # both operands of the GEMM must come from pieces of this split when both read src
                if ab == src and r.data.get("h3a") != name or bb == src and r.data.get("h3b") != name:
                    ok = False
                    break
            k.data["pieces_only"] = ok

    def _first_side_gemm(self) -> int:
        if not hasattr(self, "_fsg"):
            ks = self.comp.kernels
            self._fsg = next((i for i, k in enumerate(ks) if k.kind == "gemm" and self.stream_of.get(i)), len(ks))
        return self._fsg

    def _emit_copy(self, k):
        d = k.data
        buf = d["buf"]
        dims = self.comp.bufdims[buf] if d["dir"] == 0 else self.comp.f.result_types[d["j"]].dims
        nbytes = 4 * _prod(dims)
        for p in range(self.ndev):
            q = R.CopyParams()
            q.dev = self.addr(p, buf)
            q.host = 0
            q.bytes = nbytes
            q.dir = d["dir"]
            if d["dir"] == 0:
                self.copy_in[(buf, p)] = len(self._records)
            else:
                self.copy_out[(d["j"], p)] = len(self._records)
            self._records.append((R.K_COPY, q))

    def _emit_split(self, k):
        d = k.data
        buf, off, ld = d["src"]
        p = R.SplitParams()
        p.base, p.dev_stride, p.ndev = self.base, self.dev_stride, self.ndev
        p.rows, p.cols = d["rows"], d["cols"]
        p.src_off = self.off[buf] + off
        p.ld = ld
        p.dst_off = self.off[k.outs[0]]
        p.pitch = d["pitch"]
        p.scl_off = self.off[k.outs[0]] + d["scl_off"]
        p.flags = R.SPLIT_PIECES_ONLY if d.get("pieces_only") else 0
        self._records.append((R.K_SPLIT, p))

    # streams of a two-level schedule (runtime.cu: SPX_SIDE_STREAMS)
    MAIN, COMPUTE, COMM, UPDATE, H2D, D2H = 0, 1, 2, 3, 4, 5

    def _add_copies(self):
        """Copy kernels for the drop-in call: one H2D per argument, issued in
        the order the step first reads them (so the first block's weights
        arrive first and compute starts while later ones are in flight), one
        D2H per result right after the kernel that last writes it (parameter
        updates are hoisted next to their gradients, so most results leave
        during the backward pass)."""
        c = self.comp
        ks = c.kernels
        first_read = {}
        last_write = {}
        for i, k in enumerate(ks):
            for b in k.ins:
                first_read.setdefault(b, i)
            for b in k.outs:
                last_write[b] = i
        order = sorted(c.arg_bufs, key=lambda a: (first_read.get(a, len(ks)), c.arg_bufs.index(a)))
        ins = [Kernel("copy", [a], set(), data=dict(dir=0, buf=a)) for a in order]
        after: dict = {}
        for j, b in enumerate(c.result_bufs):
            after.setdefault(last_write.get(b, -1), []).append(Kernel("copy", [], {b}, data=dict(dir=1, buf=b, j=j)))
        out = list(ins) + after.get(-1, [])
        for i, k in enumerate(ks):
            out.append(k)
            out.extend(after.get(i, []))
        c.kernels = out

    def _terminal(self, k) -> bool:
        """A kernel whose outputs are only function results (parameter and
        momentum updates, the loss) -- nothing downstream waits for it."""
        results = set(self.comp.result_bufs)
        return k.kind in ("ew", "reduce") and all(b in results for b in k.data.get("outs_keep", k.outs))

    def _hoist_terminal(self):
        """Move every terminal kernel -- and every collective whose outputs
        only terminal kernels read -- to just after its last producer.  The
        reference's training steps emit all parameter updates (and, once
        partitioned, their gradient reductions) after the whole backward pass,
        in forward order (models.py:152-220), so as written the first update
        waits for the LAST weight gradient; hoisted, each gradient collective
        and update runs (on its own stream) as soon as its gradient exists."""
        import os
        ks = self.comp.kernels
        n = len(ks)
        readers: dict = {}
        for i, k in enumerate(ks):
            for b in k.ins:
                readers.setdefault(b, []).append(i)
        results = set(self.comp.result_bufs)
        # Gradient collectives (reduce-scatters / all-reduces whose outputs
        # feed only the updates) move too, to just after their gradient: as
        # written they all follow the backward pass, and the collective stream
        # runs collectives in order, so the first one waited for the LAST
        # gradient and the whole queue drained after the compute (C3 N=4: a
        # 9.4 ms tail of reduce-scatters, profiles/r02_timeline_n4.txt).  The
        # order stays deterministic, hence identical on every rank.
        hoist_coll = os.environ.get("SPX_HOIST_COLL", "1") != "0"
        movable = [False] * n
        for i in reversed(range(n)):
            k = ks[i]
            rd = [j for b in k.outs for j in readers.get(b, [])]
            if self._terminal(k) and not rd:
                movable[i] = True
            elif (hoist_coll and k.kind == "coll" and rd and all(movable[j] for j in rd)
                  and not any(b in results for b in k.outs)):
                movable[i] = True
        # a moved kernel is emitted right after the LAST of its producers to
        # be emitted (producers may themselves have moved)
        prod = {}
        waiters: dict = {}
        remaining = {}
        for i, k in enumerate(ks):
            if movable[i]:
                deps = {prod[b] for b in k.ins if b in prod}
                remaining[i] = len(deps)
                for d in deps:
                    waiters.setdefault(d, []).append(i)
            for b in k.outs:
                prod[b] = i
        # SPX_HOIST_YIELD=w (opt-in): a moved collective yields to the next
        # critical collective -- emitted after the next collective that stays
        # in place, or after w further kernels -- so that on the in-order
        # collective stream a gradient all-reduce does not hold back the
        # row-parallel all-reduce of the same layer (C2 N=4 timeline: ~45 us
        # per block).  Measured slower (C2 N=4 894k -> 874k, C5 853k -> 837k,
        # C3 137.9k -> 136.4k, profiles/r02_hoist_yield_n4.txt): off.
        window = int(os.environ.get("SPX_HOIST_YIELD", "0"))
        order = []
        done = set()
        deferred: list = []

        def talks(k):          # a collective that moves data between ranks / devices
            return k.kind == "coll" and k.data.get("kind") != "all_slice"

        def release(j):
            if window > 0 and talks(ks[j]):
                deferred.append([j, window])
                done.add(j)            # queued: emitted by flush()
            else:
                emit(j)

        def emit(i):
            order.append(ks[i])
            done.add(i)     # (already there for a deferred collective)
            for j in waiters.get(i, []):
                remaining[j] -= 1
                if remaining[j] == 0:
                    release(j)

        def flush(all_=True):
            while deferred and (all_ or deferred[0][1] <= 0):
                emit(deferred.pop(0)[0])

        for i in range(n):
            if movable[i] and remaining[i] == 0 and i not in done:
                release(i)
        for i in range(n):
            if movable[i]:
                continue
            emit(i)
            if talks(ks[i]):
                flush()
            else:
                for d in deferred:
                    d[1] -= 1
                flush(all_=False)
        flush()
        assert len(order) == n
        self.comp.kernels = order

    def _streams(self) -> dict:
        """Kernel index -> side stream for everything off the critical path:
        * COMM: NCCL collectives whose results feed only the parameter update
          (gradient reductions; SPX_SIDE_ALL_COLLECTIVES=1: every collective);
        * COMPUTE: off-critical-path GEMMs -- weight gradients whose results
          feed only the update or a side-stream collective (act^T @ dh in
          matmul_grads, models.py:64-71); a small-tile dW GEMM then fills SMs
          the dX GEMM leaves idle;
        * UPDATE: terminal kernels (parameter/momentum updates, the loss).
        Everything else stays in program order on the main stream."""
        import os
        c = self.comp
        ks = c.kernels
        readers: dict = {}
        for i, k in enumerate(ks):
            for b in k.ins:
                readers.setdefault(b, []).append(i)

        results = set(c.result_bufs)

        crit_coll_set = set()     # collectives on the collective stream that the critical path waits for

        def off_critical(i, side):
            rd = [j for b in ks[i].outs for j in readers.get(b, [])]
            if not rd:       # writes only results: a GEMM with a fused update
                return ks[i].kind == "gemm" and all(b in results for b in ks[i].outs)
            return all(self._terminal(ks[j]) or (j in side and j not in crit_coll_set) for j in rd)

        side: dict = {}
        crit_coll = os.environ.get("SPX_SIDE_ALL_COLLECTIVES", "0") == "1"
        prefetch = os.environ.get("SPX_PREFETCH", "1") != "0"
        # Forward progress by construction: every cross-rank
        # collective of a rank -- peer kernels and NCCL calls alike -- is issued
        # on ONE stream, in program order, identical on every rank.  A rank then
        # holds at most one spinning collective at a time, and the k-th
        # collective of every member is launched only after all its members
        # completed their earlier ones and its local producers finished (which
        # need no remote progress), so no cycle of SM residency and cross-stream
        # waits can form, whatever the compute streams run (side-stream GEMMs
        # included).  SPX_COLL_ONE_STREAM=0 restores the round-1 placement
        # (critical-path collectives on the main stream).
        one = c.comm_mode == "nccl" and os.environ.get("SPX_COLL_ONE_STREAM", "1") != "0"
        args = set(c.arg_bufs)
        self.coll_offcrit = set()     # collectives nothing on the critical path waits for
        self.crit_colls = set()       # cross-rank collectives the critical path waits for
        if c.comm_mode == "nccl":
            for i in reversed(range(len(ks))):
                k = ks[i]
                if k.kind == "coll" and k.data["kind"] != "all_slice":
                    off = off_critical(i, side) or (prefetch and k.data["kind"] == "all_gather" and k.ins
                                                    and all(b in args for b in k.ins))
                    if off:
                        self.coll_offcrit.add(i)
                    if one or crit_coll or off:
                        side[i] = self.COMM
                        if not off:
                            self.crit_colls.add(i)
                        if not off and os.environ.get("SPX_CRIT_PRODUCERS_MAIN", "1") != "0":
                            # on the collective stream only for forward progress:
                            # its producers (the row-parallel GEMM before an
                            # all-reduce) stay on the main stream
                            crit_coll_set.add(i)
        # splits of function arguments run on the compute stream from the start
        # of the step, overlapped with the forward pass (their GEMMs wait for them)
        # ... and, with SPX_PREFETCH_SPLITS=1, the splits of prefetched
        # parameter gathers (ZeRO-3), which depend only on the gather: measured
        # neutral (C3 N=4 140.3k vs 140.7k, profiles/r02_prefetch_splits_n4.txt),
        # so they stay in front of their GEMM on the main stream
        pref_split = os.environ.get("SPX_PREFETCH_SPLITS", "0") != "0"
        coll_out = {b: j for j in self.coll_offcrit for b in ks[j].outs}
        for i, k in enumerate(ks):
            if k.kind == "split" and (k.data["src"][0] in args or (pref_split and k.data["src"][0] in coll_out)):
                side[i] = self.COMPUTE
        # side-stream GEMMs (whole-SM CTAs): with every collective on one stream
        # they cannot close a cross-rank residency cycle; under the round-1
        # placement (SPX_COLL_ONE_STREAM=0) only below 4 ranks
        cg_default = "0" if c.comm_mode == "nccl" and not one and self.mesh_size >= 4 else "1"
        if os.environ.get("SPX_CONCURRENT_GEMM", cg_default) != "0":
            for i in reversed(range(len(ks))):
                # in-kernel split-K GEMMs share one workspace: main stream only
                if (ks[i].kind in ("gemm", "split") and not ks[i].data.get("sk_inkernel")
                        and off_critical(i, side)):
                    side[i] = self.COMPUTE
        if os.environ.get("SPX_UPDATE_STREAM", "1") != "0" and side:
            for i, k in enumerate(ks):
                if self._terminal(k):
                    side[i] = self.UPDATE
        for i, k in enumerate(ks):
            if k.kind == "copy":
                side[i] = self.D2H if k.data["dir"] else self.H2D
        return side

    def _schedule(self):
        """Multi-stream schedule: a record waits for the LATEST earlier record
        on each other stream whose arena intervals conflict with it (RAW, WAR
        or WAW -- the liveness packing reuses memory, so WAR/WAW matter too)."""
        c = self.comp
        iv = {}

        def ivals(names):
            out = []
            for b in names:
                o = self.off[b]
                out.append((o, o + _align(c.buffers[b])))
            return out

        kin, kout, kstream = [], [], []
        for i, k in enumerate(c.kernels):
            kstream.append(self.stream_of.get(i, self.MAIN))
            r = ivals(k.ins)
            w = ivals(k.outs)
            if k.kind == "reduce":
                sc = (self.scratch_off, self.zero_off)
                r.append(sc)
                w.append(sc)
            if k.data.get("stage"):
                # NCCL relayouts share the staging region: order
                # every collective that uses it
                st_iv = (self.stage_a, self.stage_b + self.stage_elems)
                r.append(st_iv)
                w.append(st_iv)
            kin.append(r)
            kout.append(w)

        def hit(a, b):
            return any(x0 < y1 and y0 < x1 for x0, x1 in a for y0, y1 in b)

        sched = []
        by_stream: dict = {}
        for i, k in enumerate(c.kernels):
            st = kstream[i]
            waits = []
            for o, lst in by_stream.items():
                if o == st:
                    continue
                for j in reversed(lst):
                    if hit(kin[i], kout[j]) or hit(kout[i], kin[j]) or hit(kout[i], kout[j]):
                        if self._krange[j][1] > self._krange[j][0]:
                            waits.append(self._krange[j][1] - 1)
                        break
            first, end = self._krange[i]
            for r in range(first, end):
                if st or waits:
                    sched.append((r, st, sorted(waits) if r == first else []))
            by_stream.setdefault(st, []).append(i)
        if not any(st for _, st, _ in sched):
            return []
        return sched

    def _emit_reduce(self, k):
        in_dims = list(k.data["in_dims"]) or [1]
        red = sorted(k.data["red"])
        kept = [d for d in range(len(in_dims)) if d not in red]
        root = k.data["root"]
        prog = Program.build({k.outs[0]: root})
        views = []
        for l in prog.leaves:
            st = list(l.strides) if len(l.strides) == len(in_dims) else [0] * len(in_dims)
            views.append(st)
        cst = list(_contig(in_dims))
        # collapse kept dims and reduced dims separately (views + the logical layout)
        kd, kv = _collapse([in_dims[d] for d in kept], [[v[d] for d in kept] for v in views + [cst]]) \
            if kept else ([], [[] for _ in views + [cst]])
        rd, rv = _collapse([in_dims[d] for d in red], [[v[d] for d in red] for v in views + [cst]])
        p = R.ReduceParams()
        x = p.x
        x.base, x.dev_stride, x.ndev = self.base, self.dev_stride, self.ndev
        dims = list(kd) + list(rd)
        x.rank = len(dims)
        for i, dd in enumerate(dims):
            x.dims[i] = dd
        x.numel = _prod(in_dims)
        x.n_in = len(prog.leaves)
        for j, l in enumerate(prog.leaves):
            x.inp[j].off = self.off[l.buf] + l.off
            for i, st in enumerate(list(kv[j]) + list(rv[j])):
                x.inp[j].stride[i] = st
        x.n_out = 1
        x.out_reg[0] = prog.out_regs[0]
        x.n_prog = len(prog.insns)
        for i, (op, a, b, dst, imm) in enumerate(prog.insns):
            x.prog[i].op, x.prog[i].a, x.prog[i].b, x.prog[i].dst = op, a, b, dst
            x.imm[i] = self._imm(imm)
        x.dtype = self.dt
        p.monoid = 0 if k.data["monoid"] == "sum" else 1
        p.n_kept, p.n_red = len(kd), len(rd)
        p.n_out = _prod(in_dims[d] for d in kept)
        p.n_red_elems = _prod(in_dims[d] for d in red)
        p.out_off = self.off[k.outs[0]]
        p.scratch_off = self.scratch_off
        # thread mapping: innermost logical dim reduced -> ROW, kept -> COL
        two_d = len(kd) <= 1 and len(rd) == 1
        innermost_kept = bool(kept) and kept[-1] == len(in_dims) - 1
        nl = len(prog.leaves)
        out_vec = (bool(kd) and p.n_out % 4 == 0 and kd[-1] % 4 == 0 and
                   all(kv[j][-1] in (0, 1) for j in range(nl)) and
                   all(x.inp[j].off % 4 == 0 and all(st % 4 == 0 for st in list(kv[j][:-1]) + list(rv[j]))
                       for j in range(nl) if kv[j][-1] == 1))
        if p.n_red_elems <= 64 and p.n_out >= 4096 and out_vec:
            p.mode = 3
            x.vec = 1
        elif not two_d:
            p.mode = 2
            x.vec = 0
        elif innermost_kept:
            p.mode = 1
            so = [kv[j][0] if kd else 0 for j in range(len(prog.leaves))]
            x.vec = int(p.n_out % 4 == 0 and all(s_ in (0, 1) for s_ in so) and
                        all((x.inp[j].off % 4 == 0) and (rv[j][0] % 4 == 0) for j in range(len(prog.leaves))
                            if so[j] == 1))
        else:
            p.mode = 0
            sr = [rv[j][0] for j in range(len(prog.leaves))]
            x.vec = int(p.n_red_elems % 4 == 0 and all(s_ in (0, 1) for s_ in sr) and
                        all((x.inp[j].off % 4 == 0) and (not kd or kv[j][0] % 4 == 0)
                            for j in range(len(prog.leaves)) if sr[j] == 1))
        self._records.append((R.K_REDUCE, p))

    def _emit_gemm(self, k):
        d = k.data
        p = R.GemmParams()
        p.base, p.dev_stride, p.ndev = self.base, self.dev_stride, self.ndev
        p.M, p.N, p.K = d["M"], d["N"], d["K"]
        ab, aoff, lda, at = d["a"]
        bb, boff, ldb, bt = d["b"]
        p.a_off = self.off[ab] + aoff
        p.b_off = self.off[bb] + boff
        p.c_off = self.off[k.outs[0]]
        p.lda, p.ldb, p.ldc = lda, ldb, d["N"]
        p.a_mn_major = 1 if at else 0
        p.b_k_major = 1 if bt else 0
        p.path = self.gemm_path
        p.splits = d.get("splits", 1)
        if p.splits > 1:
            p.path = 1                       # split-K partials exist on the tcgen05 path only
        if d.get("sk_inkernel"):
            p.sk_mode = 1
            p.ws_off = self.sk_ws_off
            p.flag_off = self.sk_flag_off
        epi = d.get("epi")
        if epi is not None:
            p.path = 1                       # fused epilogues exist on the tcgen05 path only
            p.epi = epi["kind"]
            for j, x in enumerate(epi["xs"]):
                p.epi_in_off[j] = self.off[x.buf] + x.off
                p.epi_in_ld[j] = x.strides[0]
            for j, o in enumerate(epi["outs"]):
                p.epi_out_off[j] = self.off[o]
                p.epi_out_ld[j] = d["N"]
            p.epi_imm[0], p.epi_imm[1] = epi["imm"]
            p.c_off = self.off[epi["outs"][0]]
        if "h3a" in d:
            p.path = 3
            p.h3_shared = 1
            # split-K (opt-in, SPX_H3_SPLITK) only while nothing else computes:
            # before the first GEMM of a side stream (the forward pass)
            p.h3_splitk = d.get("h3_splitk") or (0 if self._cur < self._first_side_gemm() else 1)
            p.h3_a_off = self.off[d["h3a"]]
            p.h3_b_off = self.off[d["h3b"]]
            p.h3_a_scl = p.h3_a_off + d["h3a_scl"]
            p.h3_b_scl = p.h3_b_off + d["h3b_scl"]
        # with collectives overlapped on a side stream, leave SMs for NCCL's CTAs
        p.reserve_sms = self.reserve_sms
        if self.stream_of.get(self._cur) == self.COMPUTE and getattr(self, "crit_colls", None):
            # a side-stream GEMM (persistent, whole-SM CTAs) would otherwise hold
            # every SM when a critical-path collective is launched next to it
            p.reserve_sms = max(p.reserve_sms, int(_os.environ.get("SPX_SIDE_GEMM_RESERVE", "0")))
        p.dtype = self.dt
        self._records.append((R.K_GEMM, p))

    # ---- in-GPU collectives (spmd_interp.py:74-123 as group kernels) ----
    def _ptrs(self, buf, extra=0):
        return np.array([self.addr(p, buf, extra) for p in range(self.ndev)], dtype=np.uint64)

    def _emit_coll_local(self, k):
        c = self.comp
        d = k.data
        kind, attrs = d["kind"], d["attrs"]
        src, out = d["src"], k.outs[0]
        in_dims, out_dims = list(d["in_dims"]), list(d["out_dims"])
        S = _contig(in_dims)
        coords = c.coords
        devs = c.devices
        assert devs == list(range(len(coords))), "local mode hosts every mesh device"
        if kind in ("all_slice", "all_gather", "all_to_all"):
            g = R.GatherParams()
            g.ndev = self.ndev
            g.rank = len(out_dims)
            g.numel = _prod(out_dims)
            for j, dd in enumerate(out_dims):
                g.dims[j] = dd
                g.sstride[j] = S[j]
            base = np.zeros(self.ndev, dtype=np.int64)
            if kind == "all_slice":
                apd = attrs["axes_per_dim"]
                for j, dd in enumerate(out_dims):
                    g.ext[j] = dd
                g.n_combo = 1
                table = np.array([self.addr(p, src) for p in range(self.ndev)], dtype=np.uint64)
                for p in range(self.ndev):
                    base[p] = sum(c._chunk_index(coords[p], apd[j]) * out_dims[j] * S[j]
                                  for j in range(len(out_dims)))
            elif kind == "all_gather":
                apd = attrs["axes_per_dim"]
                nper = [out_dims[j] // in_dims[j] for j in range(len(out_dims))]
                cm = _contig(nper)
                for j in range(len(out_dims)):
                    g.ext[j] = in_dims[j]
                    g.cmul[j] = cm[j]
                g.n_combo = _prod(nper)
                axes = [a for axs in apd for a in axs]
                grp = c._group_of(axes)
                zero = self.base + self.zero_off * 4
                table = np.full((self.ndev, g.n_combo), zero, dtype=np.uint64)
                for p in range(self.ndev):
                    for m in grp[p]:
                        combo = sum(c._chunk_index(coords[m], apd[j]) * cm[j] for j in range(len(apd)))
                        table[p, combo] = self.addr(m, src)
            else:  # all_to_all
                gd, sd, axes = attrs["gather_dim"], attrs["slice_dim"], attrs["axes"]
                n = c._axes_n(axes)
                for j, dd in enumerate(out_dims):
                    g.ext[j] = dd
                g.ext[gd] = in_dims[gd]
                g.cmul[gd] = 1
                g.n_combo = n
                grp = c._group_of(axes)
                table = np.zeros((self.ndev, n), dtype=np.uint64)
                for p in range(self.ndev):
                    for m in grp[p]:
                        table[p, c._chunk_index(coords[m], axes)] = self.addr(m, src)
                    base[p] = c._chunk_index(coords[p], axes) * out_dims[sd] * S[sd]
            g.src_table = self._tref(table.reshape(-1))
            g.base_off = self._tref(base)
            g.dst = self._tref(self._ptrs(out))
            self._records.append((R.K_GATHER, g))
            return
        # all_reduce / reduce_scatter: left fold in group order (_combine, :66-71)
        axes = attrs["axes"]
        grp = c._group_of(axes)
        nm = len(grp[0])
        r = R.CreduceParams()
        r.ndev, r.rank, r.n_members = self.ndev, len(out_dims), nm
        r.monoid = 0 if attrs.get("monoid", "sum") == "sum" else 1
        r.numel = _prod(out_dims)
        for j, dd in enumerate(out_dims):
            r.dims[j] = dd
            r.sstride[j] = S[j]
        members = np.array([grp[p] for p in range(self.ndev)], dtype=np.int32)
        base = np.zeros(self.ndev, dtype=np.int64)
        if kind == "reduce_scatter":
            apd = attrs["axes_per_dim"]
            for p in range(self.ndev):
                base[p] = sum(c._chunk_index(coords[p], apd[j]) * out_dims[j] * S[j]
                              for j in range(len(out_dims)))
        r.dtype = self.dt
        r.src = self._tref(self._ptrs(src))
        r.members = self._tref(members.reshape(-1))
        r.base_off = self._tref(base)
        r.dst = self._tref(self._ptrs(out))
        self._records.append((R.K_CREDUCE, r))

    # ---- NCCL collectives (one mesh device per process) ----
    def comm_keys(self):
        """(axes key, group) for every communicator this program needs, in a
        deterministic order shared by all ranks."""
        c = self.comp
        keys = []
        for k in c.kernels:
            if k.kind != "coll" or k.data["kind"] == "all_slice":
                continue
            a = k.data["attrs"]
            axes = a["axes"] if "axes" in a else [x for axs in a["axes_per_dim"] for x in axs]
            key = tuple(sorted(set(axes), key=c.mesh.names().index))
            if key not in keys:
                keys.append(key)
        return keys

    def _nccl(self, kind, comm, send, recv, count, monoid=0):
        if comm < 0:
            raise UnsupportedProgram("this collective needs NCCL, but no communicator exists (SPX_NCCL_NONE=1)")
        p = R.NcclParams()
        p.kind, p.comm, p.monoid = kind, comm, monoid
        p.send, p.recv, p.count = send, recv, count
        self._records.append((R.K_NCCL, p))

    def _gather1(self, out_addr, dims, ext, cmul, sstride, table, base=0):
        g = R.GatherParams()
        g.ndev, g.rank, g.numel = 1, len(dims), _prod(dims)
        for j, dd in enumerate(dims):
            g.dims[j], g.ext[j], g.cmul[j], g.sstride[j] = dd, ext[j], cmul[j], sstride[j]
        g.n_combo = len(table)
        g.src_table = self._tref(np.array(table, dtype=np.uint64))
        g.base_off = self._tref(np.array([base], dtype=np.int64))
        g.dst = self._tref(np.array([out_addr], dtype=np.uint64))
        self._records.append((R.K_GATHER, g))

    def _ar_key(self, k):
        a = k.data["attrs"]
        axes = a["axes"] if "axes" in a else [x for axs in a["axes_per_dim"] for x in axs]
        return tuple(sorted(set(axes), key=self.comp.mesh.names().index))

    def peer_slots(self):
        """Flag/epoch slots of the peer all-reduce: one per (communicator,
        stream).  Peer all-reduces on one slot run in stream order; different
        streams never share flag words, so the gradient reductions on the
        collective stream and the critical-path ones on the main stream both
        take the peer path.  Same order on every rank (same program and
        schedule).  SPX_PEER_SIDE=0: critical-path all-reduces only."""
        import os
        if not hasattr(self, "_slots"):
            slots = [(key, self.MAIN) for key in self.comm_keys()]
            if os.environ.get("SPX_PEER_SIDE", "1") != "0":
                for i, k in enumerate(self.comp.kernels):
                    if k.kind == "coll" and k.data["kind"] in ("all_reduce", "reduce_scatter", "all_gather"):
                        sk = (self._ar_key(k), self.stream_of.get(i, self.MAIN))
                        if sk not in slots:
                            slots.append(sk)
            self._slots = slots
        return self._slots

    def _peer_slot(self, key):
        st = self.stream_of.get(self._cur, self.MAIN)
        if st != self.MAIN and (key, st) not in self.peer_slots():
            return None
        return self.peer_slots().index((key, st))

    def _emit_coll_nccl(self, k):
        import os
        c = self.comp
        d = k.data
        kind, attrs = d["kind"], d["attrs"]
        me = c.devices[0]
        coords = c.coords
        src, out = d["src"], k.outs[0]
        in_dims, out_dims = list(d["in_dims"]), list(d["out_dims"])
        S = _contig(in_dims)
        src_a, out_a = self.addr(0, src), self.addr(0, out)
        sa = self.base + self.stage_a * 4
        sb = self.base + self.stage_b * 4
        if kind == "all_slice":
            apd = attrs["axes_per_dim"]
            base = sum(c._chunk_index(coords[me], apd[j]) * out_dims[j] * S[j] for j in range(len(out_dims)))
            self._gather1(out_a, out_dims, out_dims, [0] * len(out_dims), S, [src_a], base)
            return
        axes = attrs["axes"] if "axes" in attrs else [x for axs in attrs["axes_per_dim"] for x in axs]
        key = tuple(sorted(set(axes), key=c.mesh.names().index))
        grp = c._group_of(list(key))[me]
        comm = self.comms[key]
        n = len(grp)
        monoid = 0 if attrs.get("monoid", "sum") == "sum" else 1
        slot = self._peer_slot(key)
        use_peer = self.peer_bases is not None and 1 < n <= 8 and slot is not None

        def peer(pkind, count, src_shift=0):
            # off the critical path, a one-block barrier kernel first: the full
            # grid launches only once every member has arrived, so it does not
            # hold an SM on every SM while it waits for slower ranks
            if (pkind != 3 and self.peer_prebarrier and self._cur in getattr(self, "coll_offcrit", ())
                    and not getattr(self, "_in_prebarrier", False)):
                self._in_prebarrier = True
                peer(3, 0)
                self._in_prebarrier = False
            p = R.PeerParams()
            p.kind, p.n, p.me, p.monoid, p.count, p.slot = pkind, n, grp.index(me), monoid, count, slot
            for j, r in enumerate(grp):
                p.src[j] = self.peer_bases[r] + (src_a - self.base) + src_shift
                p.flags[j] = self.peer_bases[r] + self.flag_off * 4
            p.dst = out_a
            p.counter = self.base + self.counter_off * 4
            # off the critical path (ZeRO-3 parameter prefetch, gradient reductions):
            # a few blocks stream it while the GEMMs keep the other SMs
            if self._cur in getattr(self, "coll_offcrit", ()) and count * 4 * n >= self.peer_offcrit_min_bytes:
                p.max_blocks = self.peer_offcrit_blocks
            else:
                p.max_blocks = self.peer_side_blocks if (self._cur in self.side and not self.one_stream) else 0
            self._records.append((R.K_PEER, p))

        if kind == "all_reduce":
            count = _prod(in_dims)
            if use_peer and count * 4 <= self.peer_max_bytes:
                peer(0, count)
                return
            self._nccl(R.NCCL_ALLREDUCE, comm, src_a, out_a, count, monoid)
            return
        if kind == "all_gather":
            apd = attrs["axes_per_dim"]
            nloc = _prod(in_dims)
            nper = [out_dims[j] // in_dims[j] for j in range(len(out_dims))]
            cm = _contig(nper)
            combo_of = [sum(c._chunk_index(coords[m], apd[j]) * cm[j] for j in range(len(apd))) for m in grp]
            direct = (all(not apd[j] for j in range(1, len(apd))) and combo_of == list(range(n))
                      and _prod(nper) == n)
            # every direct gather: the ZeRO-3 parameter prefetch (function
            # arguments, C3/C5) and the ZeRO-2 gathers of freshly updated
            # shards at the end of the step (C4); SPX_PEER_AG_ALL=0 keeps the
            # latter on NCCL
            # gathers of function arguments (the ZeRO-3 parameter prefetch): the
            # copy engines pull every member's shard over NVLink straight into
            # the output -- no SM spins or copies, so the gather overlaps the
            # GEMMs completely; arguments are immutable during the step, so no
            # cross-rank handshake is needed (io calls barrier the ranks first)
            if (direct and self.peer_bases is not None and src in c.arg_bufs and self.ce_ag
                    and n * nloc * 4 >= self.ce_min_bytes):
                for j, r in enumerate(grp):
                    q = R.CopyParams()
                    q.dev = out_a + j * nloc * 4
                    q.host = self.peer_bases[r] + (src_a - self.base) if r != me else src_a
                    q.bytes = nloc * 4
                    q.dir = 2
                    self._records.append((R.K_COPY, q))
                return
            if (direct and use_peer and n in (2, 3, 4, 8) and nloc % 4 == 0 and n * nloc * 4 <= self.peer_max_bytes
                    and self.peer_ag and (src in c.arg_bufs or self.peer_ag_all)):
                peer(1, nloc)
                return
            if direct:
                self._nccl(R.NCCL_ALLGATHER, comm, src_a, out_a, nloc)
                return
            k.data["stage"] = True
            self._nccl(R.NCCL_ALLGATHER, comm, src_a, sa, nloc)
            table = [self.base + self.zero_off * 4] * _prod(nper)
            for j, cb in enumerate(combo_of):
                table[cb] = sa + j * nloc * 4
            self._gather1(out_a, out_dims, in_dims, cm, _contig(in_dims), table)
            return
        if kind == "reduce_scatter":
            apd = attrs["axes_per_dim"]
            nout = _prod(out_dims)
            offs = [sum(c._chunk_index(coords[m], apd[j]) * out_dims[j] * S[j] for j in range(len(apd)))
                    for m in grp]
            if offs == [j * nout for j in range(n)]:
                if use_peer and self.ce_rs and (n - 1) * nout <= self.stage_elems and n * nout * 4 >= self.ce_min_bytes:
                    # copy-engine reduce-scatter: a one-block barrier (every member's
                    # input is complete), the copy engines pull this member's chunk of
                    # every peer's input into staging, a local kernel folds the chunks
                    # in member order (the reference's _combine, bit-identical), a
                    # one-block barrier releases the inputs.  Only the two barriers
                    # wait on peers, each holding one SM instead of every SM.
                    k.data["stage"] = True
                    mi = grp.index(me)
                    peer(3, 0)
                    ptrs = []
                    for j, r in enumerate(grp):
                        if r == me:
                            ptrs.append(src_a + mi * nout * 4)
                            continue
                        dst = sa + (j - (j > mi)) * nout * 4
                        q = R.CopyParams()
                        q.dev = dst
                        q.host = self.peer_bases[r] + (src_a - self.base) + mi * nout * 4
                        q.bytes = nout * 4
                        q.dir = 2
                        self._records.append((R.K_COPY, q))
                        ptrs.append(dst)
                    r_ = R.CreduceParams()
                    r_.ndev, r_.rank, r_.n_members, r_.monoid = 1, 1, n, monoid
                    r_.numel = nout
                    r_.dims[0] = nout
                    r_.sstride[0] = 1
                    r_.dtype = self.dt
                    # src[j] = member j's chunk: member order is the fold order
                    r_.src = self._tref(np.array(ptrs, dtype=np.uint64))
                    r_.members = self._tref(np.arange(n, dtype=np.int32))
                    r_.base_off = self._tref(np.zeros(1, dtype=np.int64))
                    r_.dst = self._tref(np.array([out_a], dtype=np.uint64))
                    self._records.append((R.K_CREDUCE, r_))
                    peer(3, 0)
                    return
                if use_peer and nout % 4 == 0 and n * nout * 4 <= self.peer_max_bytes and self.peer_rs:
                    peer(2, nout, grp.index(me) * nout * 4)
                    return
                self._nccl(R.NCCL_REDUCESCATTER, comm, src_a, out_a, nout, monoid)
                return
            # relayout send buffer as [member j][chunk of member j]
            k.data["stage"] = True
            self._gather1(sa, [n] + out_dims, [1] + out_dims, [1] + [0] * len(out_dims),
                          [0] + list(S), [src_a + o * 4 for o in offs])
            self._nccl(R.NCCL_REDUCESCATTER, comm, sa, out_a, nout, monoid)
            return
        if kind == "all_to_all":
            gd, sd = attrs["gather_dim"], attrs["slice_dim"]
            piece = list(in_dims)
            piece[sd] = out_dims[sd]
            npiece = _prod(piece)
            k.data["stage"] = True
            chunk = [c._chunk_index(coords[m], list(attrs["axes"])) for m in grp]
            self._gather1(sa, [n] + piece, [1] + piece, [1] + [0] * len(piece), [0] + list(S),
                          [src_a + ch * out_dims[sd] * S[sd] * 4 for ch in chunk])
            self._nccl(R.NCCL_ALLTOALL, comm, sa, sb, npiece)
            ext = list(out_dims)
            ext[gd] = in_dims[gd]
            cmul = [0] * len(out_dims)
            cmul[gd] = 1
            table = [0] * n
            for j, ch in enumerate(chunk):
                table[ch] = sb + j * npiece * 4
            self._gather1(out_a, out_dims, ext, cmul, _contig(piece), table)
            return
        raise AssertionError(kind)

    # --------------------------------------------------------------- host I/O
    def upload_args(self, per_device: list[dict]):
        """per_device[p][arg] = local numpy array for hosted device p.  Arrays
        in pinned memory (results of an earlier call, runtime.PinnedPool) go
        by direct async DMA; pageable ones through the pinned staging ring."""
        pool = R.pinned_pool()
        for p in range(self.ndev):
            for a in self.comp.arg_bufs:
                arr = np.ascontiguousarray(per_device[p][a], dtype=self.dtype)
                if pool.contains(arr):
                    self.device.h2d(self.addr(p, a), arr)
                else:
                    self.device.h2d_staged(self.addr(p, a), arr)

    def call(self, per_device: list[dict], replay: bool) -> list[list[np.ndarray]]:
        """One step with its data movement inside the plan (io=True): bind every
        argument's page-locked host array and a fresh page-locked result array
        per result to the copy records, launch (eager, or the captured graph),
        wait.  Pageable arguments are first staged into page-locked arrays
        (multi-threaded host copy).  Returns [result j][device p]."""
        assert self.io
        pool = R.pinned_pool()
        keep = []
        for p in range(self.ndev):
            for a in self.comp.arg_bufs:
                arr = np.ascontiguousarray(per_device[p][a], dtype=self.dtype)
                if not pool.contains(arr):
                    st = pool.array(arr.shape, self.dtype)
                    if st is None:
                        raise R.BackendError("page-locked pool exhausted (SPX_PINNED_POOL_BYTES)")
                    R.call(self.device.lib.spx_host_copy, C.c_void_p(st.ctypes.data), C.c_void_p(arr.ctypes.data),
                           arr.nbytes, 16)
                    arr = st
                keep.append(arr)
                self.plan.set_host(self.copy_in[(a, p)], arr.ctypes.data)
        f = self.comp.f
        out = []
        for j in range(len(self.comp.result_bufs)):
            dims = tuple(f.result_types[j].dims)
            per = []
            for p in range(self.ndev):
                r = pool.array(dims, self.dtype)
                if r is None:
                    raise R.BackendError("page-locked pool exhausted (SPX_PINNED_POOL_BYTES)")
                self.plan.set_host(self.copy_out[(j, p)], r.ctypes.data)
                per.append(r)
            out.append(per)
        if replay:
            self.plan.replay()
        else:
            self.plan.run()
        self.device.sync()
        del keep
        return out

    def download_results(self) -> list[list[np.ndarray]]:
        """[result j][device p] local arrays."""
        f = self.comp.f
        out = []
        for j, b in enumerate(self.comp.result_bufs):
            dims = tuple(f.result_types[j].dims)
            per = []
            for p in range(self.ndev):
                a = R.pinned_pool().array(dims, self.dtype)
                if a is None:
                    a = np.empty(dims, dtype=self.dtype)
                    self.device.d2h_staged(a, self.addr(p, b))
                else:
                    self.device.d2h(a, self.addr(p, b))       # direct async DMA, one sync below
                per.append(a)
            out.append(per)
        self.device.sync()
        return out

    def run(self):
        self.plan.run()

    def records(self):
        return list(self._records)

    # ------------------------------------------------------- executed work
    ARITH = {R.OP[k] for k in ("ADD", "MUL", "NEG", "EXP", "MAX", "ADDI", "MULI", "IADD", "IMUL")}

    def _ew_flops(self, p) -> float:
        return float(sum(1 for i in range(p.n_prog) if p.prog[i].op in self.ARITH)) * p.numel * p.ndev

    def issued_per_run(self) -> dict:
        """What one run of the plan issues, derived from the records exactly as
        the runtime counts it (runtime.cu record_flops / tally_record) -- the
        CPU-side mirror used where there is no GPU (dry plans)."""
        coll = {k: 0 for k in R.COLL_ORDER}
        flops = 0.0
        epi_ops = {R.EPI_ADD: 1, R.EPI_SQUARE: 1, R.EPI_MULSCALE: 2, R.EPI_MOMENTUM: 5}
        for idx, (kind, p) in enumerate(self._records):
            tag = self._tags.get(idx, 0)
            c = tag & 7
            if c:
                coll[R.COLL_ORDER[c - 1]] += 1
            if tag & R.TAG_INTERNAL:
                continue
            if kind == R.K_GEMM:
                flops += (2.0 * p.K + epi_ops.get(p.epi, 0)) * p.M * p.N * p.ndev
            elif kind == R.K_EW:
                flops += self._ew_flops(p)
            elif kind == R.K_REDUCE:
                flops += self._ew_flops(p.x) + float(p.x.numel) * p.x.ndev
        return {"coll": coll, "flops": flops}

    def work_report(self) -> dict:
        """Executed work vs the reference simulator's prediction, per device and
        step.  `program` = collective_counts(local module) (spmd.py:264-271),
        `executed` = logical collectives the runtime issued per run (measured
        counters when the plan has run, else the record-derived count),
        `cse_elided` = collectives served by an identical earlier one (their
        executed + elided = program; SPX_COLL_CSE=0 executes every one).
        FLOPs: `simulator` = simulate().compute_flops convention (sim.py:86-100),
        `executed` = issued by the kernels, `folded` = elementwise ops with
        constant operands evaluated at compile time; executed + folded =
        simulator."""
        c = self.comp
        pred = self.issued_per_run()
        ex_coll, ex_flops, source = pred["coll"], pred["flops"], "records"
        if self.plan is not None:
            st = self.plan.exec_stats()
            if st["runs"] > 0:
                ex_coll = {k: v / st["runs"] for k, v in st["coll"].items()}
                ex_flops = st["flops"] / st["runs"]
                source = f"runtime counters over {st['runs']} runs"
        per = 1.0 / self.ndev      # FLOPs are summed over the virtual devices; a
        # collective record is one logical collective for every device group
        return {"collectives": {"program": dict(c.counts),
                                "executed": dict(ex_coll),
                                "cse_elided": dict(c.cse_elided), "source": source},
                "flops": {"simulator": c.flops, "executed": ex_flops * per, "folded": c.folded_flops}}

    def close(self):
        if self.dry:
            return
        self.plan.destroy()
        if self._own_comms:
            for cm in set(self.comms.values()):
                R.call(R.load().spx_comm_destroy, int(cm))
            self.comms = {}
            self._own_comms = False
        for ptr in self._peer_handles:
            R.call(R.load().spx_ipc_close, ptr)
        self._peer_handles = []
        self.device.free(self.base)
        self.device.free(self.table_base)
