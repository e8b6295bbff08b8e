"""Plan compiler: localized SPMD function + ShardingSpec -> device records.

This is the op-to-kernel lowering below the reference's lockstep loop
(`spmd_interpret`, /root/reference/pkg/src/spindle/spmd_interp.py:184-191).
Where the reference evaluates every op with numpy per device
(`interp._eval_op`, interp.py:35-75) and every collective as a numpy group
operation (`_run_collective`, spmd_interp.py:74-123), the compiler:

  * turns data-movement-free ops into VIEWS of buffers (transpose, broadcast,
    reshape of contiguous data, tag, all_slice of broadcast dims) or scalar
    CONSTANTS (constant and anything derived from it, folded with numpy
    float32 arithmetic so folding is bit-exact);
  * fuses chains of elementwise ops (add/mul/neg/exp) into expression
    programs -- single-use subexpressions are inlined, and producer groups
    whose consumers all run later are merged into multi-output kernels (the
    momentum update m' = 0.9 m + g; p' = p - 0.01 m' is ONE kernel);
  * folds the reduced operand of `reduce` into the reduction kernel;
  * lowers matmul to the tcgen05 3xTF32 GEMM with operand transposes folded
    into the TMA/UMMA descriptors (SIMT fallback for tiny/misaligned shapes);
  * lowers collectives either to in-GPU group kernels over co-located mesh
    devices (bit-exact left folds in group order) or to NCCL calls when each
    mesh device is its own process/GPU;
  * assigns arena offsets by liveness (cf. sim.peak_live_bytes, sim.py:126-150).

Every per-device program is identical (SPMD), so buffers sit at the same
offset in every device's arena slice and one launch covers all co-located
devices.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import runtime as R
from .ir import COLLECTIVE_KINDS, COUNTED_COLLECTIVES, op_flops

ALIGN = 64  # elements (256 B)
EW_KINDS = ("add", "mul", "neg", "exp")


def _prod(xs):
    n = 1
    for x in xs:
        n *= int(x)
    return n


def _contig(dims):
    st, acc = [], 1
    for d in reversed(dims):
        st.append(acc)
        acc *= int(d)
    return tuple(reversed(st))


def _align(n, a=ALIGN):
    return (n + a - 1) // a * a


# --- value descriptors --------------------------------------------------------

@dataclass(frozen=True)
class Leaf:
    buf: str          # buffer name
    off: int          # element offset within the buffer
    strides: tuple    # per dim of the consuming shape


@dataclass
class Node:
    """Expression node: op in EW_KINDS, children are Node | Leaf | np.float32."""
    op: str
    kids: list
    uid: int = 0


@dataclass
class Desc:
    kind: str                 # "buf" | "view" | "const" | "expr"
    dims: tuple
    buf: str | None = None    # buf / view source buffer
    off: int = 0
    strides: tuple = ()
    value: np.float32 | None = None
    node: Node | Leaf | None = None


@dataclass
class Kernel:
    kind: str                 # "ew" | "reduce" | "gemm" | "coll"
    outs: list                # buffer names written
    ins: set = field(default_factory=set)   # buffer names read
    data: dict = field(default_factory=dict)
    op_index: int = -1
    alive: bool = True


class UnsupportedProgram(NotImplementedError):
    pass


class Compiler:
    """Builds the kernel list and buffer table for one localized function.

    devices: mesh device indices hosted by this process ([all] for the
    in-GPU mode, [rank] for the one-process-per-GPU NCCL mode).
    """

    def __init__(self, module, func="main", devices=None, comm_mode="local", dtype=np.float32, h3=False):
        self.module = module
        self.h3 = h3              # GEMMs run on the block-scaled 3xFP16 kernel (gemm_h3.cu)
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.dtype(np.float32), np.dtype(np.int32)):
            raise TypeError(f"compute type {self.dtype}: the backend computes float32 or int32")
        self.is_int = self.dtype == np.dtype(np.int32)
        self.f = module.func(func)
        self.mesh = module.mesh
        n_mesh = self.mesh.device_count if self.mesh is not None else 1
        self.devices = list(range(n_mesh)) if devices is None else list(devices)
        self.coords = self.mesh.coords() if self.mesh is not None else [{}]
        self.comm_mode = comm_mode
        self.types = {}
        self.desc: dict[str, Desc] = {}
        self.buffers: dict[str, int] = {}      # name -> numel
        self.bufdims: dict[str, tuple] = {}
        self.kernels: list[Kernel] = []
        self._coll_cse: dict = {}
        self._uid = 0
        self._tmp = 0
        self.arg_bufs = []
        self.result_bufs = []
        self.counts = {k: 0 for k in COUNTED_COLLECTIVES}
        self.flops = 0.0
        # work the program lists that no kernel executes: collectives reused
        # from an identical earlier one (CSE; SPX_COLL_CSE=0 disables it) and
        # elementwise ops folded at compile time (constant operands only)
        self.cse_elided = {k: 0 for k in COUNTED_COLLECTIVES}
        self.folded_flops = 0.0
        import os
        self.coll_cse = os.environ.get("SPX_COLL_CSE", "1") != "0"
        self._matcache = {}

    # ---------------------------------------------------------------- helpers
    def _new_buf(self, dims, hint="t"):
        self._tmp += 1
        name = f"%{hint}#{self._tmp}"
        self.buffers[name] = max(1, _prod(dims))
        self.bufdims[name] = tuple(dims)
        return name

    def _node(self, op, kids):
        self._uid += 1
        return Node(op, kids, self._uid)

    def _leaf_of(self, d: Desc):
        if d.kind == "buf":
            return Leaf(d.buf, 0, _contig(d.dims))
        if d.kind == "view":
            return Leaf(d.buf, d.off, tuple(d.strides))
        if d.kind == "const":
            return d.value
        return d.node

    def _uses(self):
        uses: dict[str, list] = {}
        for i, op in enumerate(self.f.ops):
            for j, o in enumerate(op.operands):
                uses.setdefault(o, []).append((i, op))
        for r in self.f.results:
            uses.setdefault(r, []).append((len(self.f.ops), None))
        return uses

    # ------------------------------------------------------- materialization
    def materialize(self, name: str) -> str:
        """Contiguous buffer holding value `name` (emits a copy/fill if needed)."""
        d = self.desc[name]
        if d.kind == "buf":
            return d.buf
        if name in self._matcache:
            return self._matcache[name]
        out = self._new_buf(d.dims, "m")
        self._emit_ew({out: self._leaf_of(d)}, d.dims)
        self._matcache[name] = out
        return out

    def _emit_ew(self, outputs: dict, dims, op_index=-1):
        k = Kernel("ew", list(outputs), data={"exprs": dict(outputs), "dims": tuple(dims)},
                   op_index=op_index)
        k.ins = self._expr_bufs(list(outputs.values()))
        self.kernels.append(k)
        return k

    def _expr_bufs(self, roots):
        seen, out = set(), set()

        def walk(x):
            if isinstance(x, Leaf):
                out.add(x.buf)
            elif isinstance(x, Node):
                if x.uid in seen:
                    return
                seen.add(x.uid)
                for c in x.kids:
                    walk(c)
        for r in roots:
            walk(r)
        return out

    # ------------------------------------------------------------------ main
    def compile(self):
        f = self.f
        # the arithmetic type is the inputs' (np.result_type, spmd_interp.py:173),
        # not the IR's element kind: both kinds are 4 bytes (ir.py:14)
        for n, t in f.args:
            self.types[n] = tuple(t.dims)
            self.buffers[n] = max(1, _prod(t.dims))
            self.bufdims[n] = tuple(t.dims)
            self.desc[n] = Desc("buf", tuple(t.dims), buf=n)
            self.arg_bufs.append(n)
        uses = self._uses()
        for i, op in enumerate(f.ops):
            for r, t in zip(op.results, op.result_types):
                self.types[r] = tuple(t.dims)
            self._lower(i, op, uses)
            if op.kind not in COLLECTIVE_KINDS:
                self.flops += op_flops(op, [self.types[o] for o in op.operands])
            if op.kind in self.counts:
                self.counts[op.kind] += 1
        for r in f.results:
            self.result_bufs.append(self.materialize(r))
        self._merge_ew()
        self._fuse_epilogues()
        return self

    def _lower(self, i, op, uses):
        k = op.kind
        r = op.results[0] if op.results else None
        dims = tuple(op.result_types[0].dims) if op.result_types else ()
        D = self.desc
        if k == "constant":
            # np.full(dims, value, cdtype) (interp.py:39-41): the value cast by numpy itself
            D[r] = Desc("const", dims, value=np.full((1,), op.attrs["value"], dtype=self.dtype)[0])
            return
        if k == "tag":
            D[r] = D[op.operands[0]]
            return
        if k in EW_KINDS:
            if k == "exp" and self.is_int:
                raise TypeError("exp of int32 computes in float64 in the reference (np.exp); "
                                "the backend computes float32 or int32")
            kids = [self._leaf_of(D[o]) for o in op.operands]
            if all(_is_const(c) for c in kids):          # constant folding (numpy's own arithmetic)
                with np.errstate(all="ignore"):
                    a = np.array(kids, dtype=self.dtype)
                    if k == "add":
                        v = (a[:1] + a[1:2])[0]
                    elif k == "mul":
                        v = (a[:1] * a[1:2])[0]
                    elif k == "neg":
                        v = (-a[:1])[0]
                    else:
                        v = np.exp(a[:1])[0]
                D[r] = Desc("const", dims, value=v)
                self.folded_flops += op_flops(op, [self.types[o] for o in op.operands])
                return
            node = self._node(k, kids)
            u = uses.get(r, [])
            inline = (len(u) == 1 and u[0][1] is not None and
                      (u[0][1].kind in EW_KINDS or u[0][1].kind == "reduce"))
            if inline:
                D[r] = Desc("expr", dims, node=node)
            else:
                out = self._new_buf(dims, "v")
                self._emit_ew({out: node}, dims, op_index=i)
                D[r] = Desc("buf", dims, buf=out)
            return
        if k == "transpose":
            x = D[op.operands[0]]
            perm = op.attrs["perm"]
            if x.kind == "const":
                D[r] = Desc("const", dims, value=x.value)
                return
            src = x if x.kind in ("buf", "view") else self.desc_of_buf(self.materialize(op.operands[0]))
            st = src.strides if src.kind == "view" else _contig(src.dims)
            D[r] = Desc("view", dims, buf=src.buf, off=src.off if src.kind == "view" else 0,
                        strides=tuple(st[p] for p in perm))
            return
        if k == "broadcast":
            x = D[op.operands[0]]
            if x.kind == "const":
                D[r] = Desc("const", dims, value=x.value)
                return
            if x.kind == "expr":
                x = self.desc_of_buf(self.materialize(op.operands[0]))
            st_x = x.strides if x.kind == "view" else _contig(x.dims)
            st = [0] * len(dims)
            for j, dd in enumerate(op.attrs["dims"]):
                st[dd] = st_x[j]
            D[r] = Desc("view", dims, buf=x.buf, off=x.off if x.kind == "view" else 0, strides=tuple(st))
            return
        if k == "reshape":
            x = D[op.operands[0]]
            if x.kind == "const":
                D[r] = Desc("const", dims, value=x.value)
                return
            if x.kind == "view" and tuple(x.strides) == _contig(x.dims):
                D[r] = Desc("view", dims, buf=x.buf, off=x.off, strides=_contig(dims))
                return
            b = self.materialize(op.operands[0])
            D[r] = Desc("view", dims, buf=b, off=0, strides=_contig(dims))
            return
        if k == "matmul":
            self._lower_matmul(i, op, dims)
            return
        if k == "reduce":
            self._lower_reduce(i, op, dims)
            return
        if k in COLLECTIVE_KINDS:
            self._lower_collective(i, op, dims)
            return
        raise UnsupportedProgram(f"op {k!r} has no dense semantics; lower and use spmd_interpret")

    def desc_of_buf(self, b):
        return Desc("buf", self.bufdims[b], buf=b)

    # ----------------------------------------------------------------- matmul
    def _mm_operand(self, name, dims):
        d = self.desc[name]
        if d.kind == "buf":
            return d.buf, 0, dims[1], False
        if d.kind == "view":
            s0, s1 = d.strides
            if s1 == 1 and s0 >= dims[1]:
                return d.buf, d.off, s0, False
            if s0 == 1 and s1 >= dims[0]:
                return d.buf, d.off, s1, True
        b = self.materialize(name)
        return b, 0, dims[1], False

    def _lower_matmul(self, i, op, dims):
        a_dims = self.types[op.operands[0]]
        b_dims = self.types[op.operands[1]]
        ab, aoff, lda, at = self._mm_operand(op.operands[0], a_dims)
        bb, boff, ldb, bt = self._mm_operand(op.operands[1], b_dims)
        out = self._new_buf(dims, "mm")
        M, K = a_dims
        N = b_dims[1]
        splits = 1 if self.is_int else self._splitk(M, N, K, aoff, lda, boff, ldb)
        sk = self._splitk_inkernel(M, N, K, aoff, lda, boff, ldb) if splits == 1 and not at and not self.is_int else 1
        h3sk = self._h3_splitk(M, N, K, aoff, lda, boff, ldb) if splits > 1 and self.h3 else 1
        if h3sk > 1:
            # few-tile long-K GEMM (weight gradients, K = N*H*W): the 3xFP16
            # kernel splits K in-kernel (the last unit of a tile folds the
            # partials in split order) and reads the operands' shared fp16
            # pieces -- no workspace reduction launch, no tf32 operand passes
            self.kernels.append(Kernel("gemm", [out], {ab, bb}, op_index=i,
                                       data=dict(M=M, N=N, K=K, a=(ab, aoff, lda, at), b=(bb, boff, ldb, bt),
                                                 splits=1, h3_splitk=h3sk, tc_ok=True)))
        elif sk > 1:
            # few-tile activation GEMM on the critical path: partials reduced
            # inside the kernel (no workspace reduction launch)
            self.kernels.append(Kernel("gemm", [out], {ab, bb}, op_index=i,
                                       data=dict(M=M, N=N, K=K, a=(ab, aoff, lda, at), b=(bb, boff, ldb, bt),
                                                 splits=sk, sk_inkernel=True, tc_ok=True)))
        elif splits == 1:
            k = Kernel("gemm", [out], {ab, bb}, op_index=i,
                       data=dict(M=M, N=N, K=K, a=(ab, aoff, lda, at), b=(bb, boff, ldb, bt), splits=1,
                                 tc_ok=not self.is_int and self._tc_ok(M, N, K, aoff, lda, boff, ldb)))
            self.kernels.append(k)
        else:
            # split-K: partial products into a [splits, M, N] workspace, summed
            # in a fixed order by a reduction (deterministic)
            ws = self._new_buf((splits, M, N), "ws")
            self.kernels.append(Kernel("gemm", [ws], {ab, bb}, op_index=i,
                                       data=dict(M=M, N=N, K=K, a=(ab, aoff, lda, at),
                                                 b=(bb, boff, ldb, bt), splits=splits)))
            root = Leaf(ws, 0, _contig((splits, M, N)))
            self.kernels.append(Kernel("reduce", [out], {ws}, op_index=i,
                                       data=dict(root=root, in_dims=(splits, M, N), red=[0],
                                                 monoid="sum", internal=True)))
        self.desc[op.results[0]] = Desc("buf", dims, buf=out)

    NUM_SMS = 148

    @staticmethod
    def _tc_ok(M, N, K, aoff, lda, boff, ldb) -> bool:
        """The runtime's tcgen05 eligibility (gemm_tc.cu: spx_gemm_tc_supported)."""
        return (M >= 64 and N >= 32 and K >= 32 and aoff % 4 == 0 and boff % 4 == 0
                and lda % 4 == 0 and ldb % 4 == 0)

    def _splitk_inkernel(self, M, N, K, aoff, lda, boff, ldb) -> int:
        """Split count for the in-kernel split-K of an activation GEMM whose
        256 x 128 tiles occupy at most half the SMs.  Every (tile, split) unit
        must be co-resident: the split-0 CTAs wait for the others (gemm_tc.cu).
        The split-0 CTAs bring the partials in with bulk tensor loads into
        their idle TMA ring and fold them in split order.  Off by default
        (SPX_SPLITK_INKERNEL=1 enables).  Measured (graph replay): a
        1024x(1024|512) MP GEMM chain 15.5 -> 14.4 us per GEMM, 1024x1024x2048
        27.1 -> 22.2 us; whole steps: C2 N=2 3.77 -> 3.64 ms, but C2 N=4 3.71 ->
        3.85 and C5 N=4 4.00 -> 4.27 ms (the split units take the SMs the
        side-stream GEMMs and collectives overlap on)."""
        import os
        if os.environ.get("SPX_SPLITK_INKERNEL", "0") == "0":
            return 1
        if not self._tc_ok(M, N, K, aoff, lda, boff, ldb) or M % 32 or N % 4:
            return 1
        pairs = -(-M // 256) * -(-N // 128) * len(self.devices)
        nk = -(-K // 32)
        if pairs * 2 * 2 > self.NUM_SMS or nk < 16:
            return 1
        # the split-0 CTAs stage (S-1) partial 128x128 tiles in their idle TMA
        # ring (144 KB): S <= 3
        return max(1, min(3, nk // 8, (self.NUM_SMS // 2) // pairs))

    def _h3_splitk(self, M, N, K, aoff, lda, boff, ldb) -> int:
        """In-kernel split count for the 3xFP16 kernel, or 1 when its split-K
        does not apply (gemm_h3.cu h3_shape: BN = 128 tiles, N % 128 == 0,
        M % 32 == 0, the tiles fill at most half the CTA pairs, >= 2 chunks of
        128 per unit)."""
        import os
        # opt-in: measured slower than the 3xTF32 workspace split on the U-Net
        # analog's weight gradients (512x256x131072 ...: 3 GEMMs 0.2 -> 0.64 ms,
        # profiles/r02_h3_longk_c4.txt) -- operand-stream bound at 1.3 TB/s
        if os.environ.get("SPX_H3_LONGK", "0") == "0":
            return 1
        if any(v % 4 for v in (aoff, lda, boff, ldb)) or M < 64 or N % 128 or M % 32:
            return 1
        pairs = self.NUM_SMS // 2
        tiles = -(-M // 256) * (N // 128) * len(self.devices)
        nch = -(-K // 128)
        if tiles * 2 > pairs or nch < 4:
            return 1
        return max(1, min(pairs // tiles, nch // 2))

    def _splitk(self, M, N, K, aoff, lda, boff, ldb) -> int:
        """Split K when the output has too few 128x128 tiles to fill the SMs
        (weight gradients: K = batch or N*H*W) and the tcgen05 path applies."""
        if not self._tc_ok(M, N, K, aoff, lda, boff, ldb):
            return 1
        # SM units: the tcgen05 kernel computes 256 x 128 tiles on CTA pairs
        units = -(-M // 256) * 2 * -(-N // 128) * len(self.devices)
        nk = -(-K // 32)
        # split only when the tiles leave most SMs idle (F: SPX_SPLITK_F);
        # moderately small GEMMs often run concurrently on the side stream
        import os
        f = int(os.environ.get("SPX_SPLITK_F", "8"))
        if units * f > self.NUM_SMS or nk < 16:
            return 1
        s = min(nk // 8, self.NUM_SMS // units)
        return max(1, s)

    # ----------------------------------------------------------------- reduce
    def _lower_reduce(self, i, op, dims):
        if self.is_int and op.attrs.get("monoid", "sum") == "sum":
            raise TypeError("reduce sum of int32 widens to int64 in the reference (np.sum); "
                            "the backend computes float32 or int32")
        x = self.desc[op.operands[0]]
        in_dims = self.types[op.operands[0]]
        root = self._leaf_of(x)
        out = self._new_buf(dims, "red")
        k = Kernel("reduce", [out], op_index=i,
                   data=dict(root=root, in_dims=tuple(in_dims), red=list(op.attrs["dims"]),
                             monoid=op.attrs.get("monoid", "sum")))
        k.ins = self._expr_bufs([root])
        self.kernels.append(k)
        self.desc[op.results[0]] = Desc("buf", dims, buf=out)

    # ------------------------------------------------------------ collectives
    def _chunk_index(self, coord, axes):
        idx = 0
        for ax in axes:
            idx = idx * self.mesh.size(ax) + coord[ax]
        return idx

    def _axes_n(self, axes):
        return _prod(self.mesh.size(a) for a in axes)

    def _groups(self, axes):
        others = [n for n in self.mesh.names() if n not in axes]
        out: dict = {}
        for i, c in enumerate(self.coords):
            out.setdefault(tuple(c[n] for n in others), []).append(i)
        return list(out.values())

    def _group_of(self, axes):
        g = {}
        for grp in self._groups(axes):
            for d in grp:
                g[d] = grp
        return g

    def _lower_collective(self, i, op, dims):
        k = op.kind
        r = op.results[0]
        src_name = op.operands[0]
        x = self.desc[src_name]
        in_dims = tuple(self.types[src_name])
        if k == "all_slice":
            apd = op.attrs["axes_per_dim"]
            if x.kind == "const":
                self.desc[r] = Desc("const", dims, value=x.value)
                return
            sliced = [dd for dd, axes in enumerate(apd) if axes]
            if x.kind == "view" and all(x.strides[dd] == 0 for dd in sliced):
                self.desc[r] = Desc("view", dims, buf=x.buf, off=x.off, strides=x.strides)
                return
        # identical collectives of the same (immutable) buffer -- e.g. the
        # forward and backward ZeRO-3 all-gathers of a parameter -- compute
        # identical values: reuse the first result (bit-exact data movement)
        import json as _json
        cse_key = None
        if not self.coll_cse:
            pass
        elif x.kind == "buf":
            cse_key = (k, x.buf, _json.dumps(op.attrs, sort_keys=True), tuple(dims))
            hit = self._coll_cse.get(cse_key)
            if hit is not None:
                self.desc[r] = Desc("buf", dims, buf=hit)
                if k in self.cse_elided:
                    self.cse_elided[k] += 1
                return
        elif x.kind == "view" and k == "all_gather" and x.off == 0:
            # all_gather of a transposed buffer (the backward pass's W^T) is the
            # transposed view of the buffer's own all-gather, when that exists
            bd = tuple(self.bufdims.get(x.buf, ()))
            cs = _contig(bd)
            perm = []
            for j, st in enumerate(x.strides):
                cand = [q for q in range(len(bd)) if cs[q] == st and bd[q] == in_dims[j] and q not in perm]
                if not cand or (bd[cand[0]] == 1):
                    perm = None
                    break
                perm.append(cand[0])
            if perm is not None and len(perm) == len(bd) and sorted(perm) == list(range(len(bd))):
                apd = op.attrs["axes_per_dim"]
                apd_b = [None] * len(bd)
                gd = [0] * len(bd)
                for j, q in enumerate(perm):
                    apd_b[q] = apd[j]
                    gd[q] = dims[j]
                attrs_b = dict(op.attrs)
                attrs_b["axes_per_dim"] = apd_b
                hit = self._coll_cse.get((k, x.buf, _json.dumps(attrs_b, sort_keys=True), tuple(gd)))
                if hit is not None:
                    gcs = _contig(gd)
                    self.desc[r] = Desc("view", tuple(dims), buf=hit, off=0,
                                        strides=tuple(gcs[q] for q in perm))
                    self.cse_elided[k] += 1
                    return
        src = self.materialize(src_name)
        out = self._new_buf(dims, "c")
        if cse_key is not None:
            self._coll_cse[cse_key] = out
        kern = Kernel("coll", [out], {src}, op_index=i,
                      data=dict(kind=k, attrs=dict(op.attrs), in_dims=in_dims, out_dims=tuple(dims),
                                src=src))
        self.kernels.append(kern)
        self.desc[r] = Desc("buf", dims, buf=out)

    # ----------------------------------------------------- GEMM epilogues
    def _fuse_epilogues(self):
        """Fold the elementwise consumer of a GEMM output into the GEMM's
        epilogue (residual add, square activation and its backward, the
        momentum update of a weight gradient): the accumulator rows are
        transformed before they leave the SM, so the product is never written
        and re-read.  Off by default (SPX_EPILOGUE=1 enables): measured on the
        C2 step, the separate elementwise kernels -- HBM-bound, overlapped with
        the GEMMs by PDL and the side streams -- cost less than the epilogue's
        extra work on the 4 drain warps (their input loads cannot reach HBM
        bandwidth with so little memory-level parallelism per SM).  See
        DESIGN.md, "GEMM epilogue fusion"."""
        import os
        if os.environ.get("SPX_EPILOGUE", "0") == "0" or self.is_int:
            return
        kinds = {int(x) for x in os.environ.get("SPX_EPILOGUE_KINDS", "1,2,3,4").split(",") if x}
        ks = self.kernels
        readers: dict = {}
        producer = {}
        for idx, k in enumerate(ks):
            for b in k.ins:
                readers.setdefault(b, []).append(idx)
            for b in k.outs:
                producer[b] = idx
        results = set(self.result_bufs)
        for gi, G in enumerate(ks):
            if G.kind != "gemm" or G.data.get("splits", 1) != 1 or not G.data.get("tc_ok"):
                continue
            C = G.outs[0]
            M, N = G.data["M"], G.data["N"]
            rd = sorted(r for r in readers.get(C, []) if ks[r].alive)
            if not rd or ks[rd[0]].kind != "ew" or tuple(ks[rd[0]].data["dims"]) != (M, N):
                continue
            E = ks[rd[0]]
            outs = list(E.data.get("outs_keep", E.outs))
            m = _match_epilogue(E.data["exprs"], outs, C, M, N)
            if m is None:
                continue
            epi, xs, imm, gouts = m
            if epi not in kinds:
                continue
            keep_c = C in results or len(rd) > 1
            if keep_c and epi != R.EPI_SQUARE:
                continue
            if any(producer.get(x.buf, -1) > gi for x in xs):
                continue                   # an input is produced after the GEMM
            G.data["epi"] = dict(kind=epi, xs=xs, imm=imm, outs=gouts)
            G.outs = list(gouts)
            G.ins = set(G.ins) | {x.buf for x in xs}
            E.alive = False
            for b in gouts:
                producer[b] = gi
            for x in xs:
                readers.setdefault(x.buf, []).append(gi)
        self.kernels = [k for k in ks if k.alive]

    # ------------------------------------------------------ multi-output merge
    def _merge_ew(self):
        """Merge an EW kernel into a later EW kernel that reads one of its outputs
        when every other reader of the producer's outputs runs after the
        consumer (so computing the producer late is safe)."""
        ks = self.kernels
        readers: dict[str, list[int]] = {}
        for idx, kk in enumerate(ks):
            for b in kk.ins:
                readers.setdefault(b, []).append(idx)
        result_set = set(self.result_bufs)
        producer = {}
        for idx, kk in enumerate(ks):
            for b in kk.outs:
                producer[b] = idx
        for xi, X in enumerate(ks):
            if X.kind != "ew" or not X.alive:
                continue
            changed = True
            while changed:
                changed = False
                for b in sorted(X.ins):
                    yi = producer.get(b)
                    if yi is None or yi >= xi:
                        continue
                    Y = ks[yi]
                    if Y.kind != "ew" or not Y.alive or Y.data["dims"] != X.data["dims"]:
                        continue
                    ok = True
                    for ob in Y.outs:
                        for rd in readers.get(ob, []):
                            if rd != xi and rd != yi and rd <= xi and ks[rd].alive:
                                ok = False
                    if not ok:
                        continue
                    # substitute leaves of Y's outputs in X by Y's expression roots
                    sub = {ob: Y.data["exprs"][ob] for ob in Y.outs}
                    dims = X.data["dims"]
                    new_exprs = {}
                    memo = {}
                    for ob, e in X.data["exprs"].items():
                        new_exprs[ob] = _substitute(e, sub, _contig(dims), memo)
                    merged = dict(sub)
                    merged.update(new_exprs)
                    if not _fits(merged):
                        continue
                    X.data["exprs"] = merged
                    X.outs = list(merged)
                    X.ins = self._expr_bufs(list(merged.values()))
                    Y.alive = False
                    for ob in Y.outs:
                        producer[ob] = xi
                    for bb in X.ins:
                        readers.setdefault(bb, []).append(xi)
                    changed = True
                    break
        # drop outputs nobody reads any more (internal registers only)
        for xi, X in enumerate(ks):
            if X.kind != "ew" or not X.alive or len(X.outs) == 1:
                continue
            keep = [ob for ob in X.outs if ob in result_set or
                    any(rd != xi and ks[rd].alive for rd in readers.get(ob, []))]
            if not keep:
                keep = X.outs[-1:]
            X.data["outs_keep"] = keep
        self.kernels = [kk for kk in ks if kk.alive]


def _is_const(e):
    return isinstance(e, (np.float32, np.int32, float))


def _match_epilogue(exprs: dict, outs: list, C: str, M: int, N: int):
    """Recognise the elementwise consumer of a GEMM output C as one of the
    fused epilogues (include/spindle_b200.h, spx_epilogue).  Returns
    (epi, [input leaves], [imm], [output buffers]) or None.  Only exact
    structural matches: the fused kernel performs the same IEEE operations
    in the same association (add/mul operand order is immaterial -- IEEE
    addition and multiplication are commutative)."""
    def is_c(e):
        return isinstance(e, Leaf) and e.buf == C and e.off == 0 and tuple(e.strides) == (N, 1)

    def is_x(e):
        return (isinstance(e, Leaf) and e.buf != C and len(e.strides) == 2 and e.strides[1] == 1
                and e.off % 4 == 0 and e.strides[0] % 4 == 0)

    def node(e, op):
        return isinstance(e, Node) and e.op == op

    def pair(e, op, f, g):
        """e = op(a, b) with f(a) and g(b) in either order -> (a, b) or None."""
        if not node(e, op) or len(e.kids) != 2:
            return None
        a, b = e.kids
        if f(a) and g(b):
            return a, b
        if f(b) and g(a):
            return b, a
        return None

    def scaled(e):
        """e = x * k (either order) -> (x leaf, k) or None."""
        m = pair(e, "mul", is_x, _is_const)
        return (m[0], float(m[1])) if m else None

    if len(outs) == 1:
        e = exprs[outs[0]]
        m = pair(e, "add", is_c, is_x)
        if m:
            return R.EPI_ADD, [m[1]], [0.0, 0.0], [outs[0]]
        if node(e, "mul") and len(e.kids) == 2 and is_c(e.kids[0]) and is_c(e.kids[1]):
            return R.EPI_SQUARE, [], [0.0, 0.0], [C, outs[0]]
        m = pair(e, "mul", is_c, lambda q: scaled(q) is not None)
        if m:
            x, k = scaled(m[1])
            return R.EPI_MULSCALE, [x], [k, 0.0], [outs[0]]
        return None
    if len(outs) == 2:
        for mo, po in ((outs[0], outs[1]), (outs[1], outs[0])):
            em, ep = exprs[mo], exprs[po]
            m = pair(em, "add", lambda q: scaled(q) is not None, is_c)
            if not m:
                continue
            mx, k0 = scaled(m[0])
            # p' = P + -(m' * k1)
            pp = pair(ep, "add", is_x, lambda q: node(q, "neg"))
            if not pp:
                continue
            inner = pp[1].kids[0]
            mm = pair(inner, "mul", lambda q: q is em or q == em, _is_const)
            if not mm:
                continue
            return R.EPI_MOMENTUM, [mx, pp[0]], [k0, float(mm[1])], [mo, po]
    return None


def _substitute(e, sub, contig, memo):
    if isinstance(e, Leaf):
        if e.buf in sub and e.off == 0 and tuple(e.strides) == tuple(contig):
            return sub[e.buf]
        return e
    if isinstance(e, Node):
        if e.uid in memo:
            return memo[e.uid]
        n = Node(e.op, [_substitute(c, sub, contig, memo) for c in e.kids], e.uid)
        memo[e.uid] = n
        return n
    return e


def _fits(exprs) -> bool:
    try:
        prog = Program.build(exprs)
    except ValueError:
        return False
    return len(prog.leaves) <= R.MAX_IN and len(prog.insns) <= R.MAX_PROG and len(exprs) <= R.MAX_OUT


class Program:
    """Expression DAG -> register-machine bytecode (spx_insn).

    Leaves (input views) are preloaded into slots 0..n_in-1; every operation
    writes a slot chosen by a liveness-based allocator over SPX_NREG slots, so
    long chains run in a fixed small register file (interp.cuh)."""

    def __init__(self):
        self.leaves: list[Leaf] = []
        self.insns: list[tuple] = []   # (op, a_slot, b_slot, dst_slot, imm)
        self.out_regs: list[int] = []

    @staticmethod
    def build(exprs) -> "Program":
        p = Program()
        memo = {}
        ssa = []          # (op, a, b, imm) with a/b = ("in", j) | ("t", i)

        def leaf(l):
            if l not in p.leaves:
                p.leaves.append(l)
            return ("in", p.leaves.index(l))

        def emit(op, a=None, b=None, imm=0.0):
            ssa.append((op, a, b, float(imm)))
            return ("t", len(ssa) - 1)

        def val(x):
            if isinstance(x, Leaf):
                return leaf(x)
            if _is_const(x):
                return emit(R.OP["IMM"], None, None, x)
            if x.uid in memo:
                return memo[x.uid]
            if x.op in ("add", "mul"):
                a, b = x.kids
                ca, cb = _is_const(a), _is_const(b)
                if cb and not ca:
                    r = emit(R.OP["ADDI" if x.op == "add" else "MULI"], val(a), None, b)
                elif ca and not cb:
                    r = emit(R.OP["IADD" if x.op == "add" else "IMUL"], val(b), None, a)
                else:
                    va, vb = val(a), val(b)
                    r = emit(R.OP["ADD" if x.op == "add" else "MUL"], va, vb)
            elif x.op == "neg":
                r = emit(R.OP["NEG"], val(x.kids[0]))
            elif x.op == "exp":
                r = emit(R.OP["EXP"], val(x.kids[0]))
            else:
                raise ValueError(x.op)
            memo[x.uid] = r
            return r

        outs = [val(e) for e in (exprs.values() if isinstance(exprs, dict) else exprs)]
        n_in = len(p.leaves)
        if n_in > R.MAX_IN or len(ssa) > R.MAX_PROG:
            raise ValueError("expression too large")
        # liveness: last instruction index reading each value; outputs live to the end
        last = {}
        for i, (op, a, b, _) in enumerate(ssa):
            for v in (a, b):
                if v is not None:
                    last[v] = i
        for v in outs:
            last[v] = len(ssa)
        slot = {("in", j): j for j in range(n_in)}
        free = [k for k in range(n_in, R.NREG)]
        for j in range(n_in):                      # inputs dead from the start
            if ("in", j) not in last:
                free.append(j)
        for i, (op, a, b, imm) in enumerate(ssa):
            for v in (a, b):                       # operands whose last use is here
                if v is not None and last.get(v) == i and slot[v] not in free:
                    free.append(slot[v])
            if ("t", i) not in last:               # dead result (cannot happen for roots)
                last[("t", i)] = i
            if not free:
                raise ValueError("expression needs more than SPX_NREG live values")
            free.sort()
            d = free.pop(0)
            slot[("t", i)] = d
            if last[("t", i)] == i:
                free.append(d)
            sa = slot[a] if a is not None else 0
            sb = slot[b] if b is not None else 0
            p.insns.append((op, sa, sb, d, imm))
        p.out_regs = [slot[v] for v in outs]
        return p
