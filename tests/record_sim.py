"""CPU simulator of the native plan records (test infrastructure only).

Executes the records an `Executable(dry=True)` emits against a numpy model of
the device arena, following the kernel contracts in include/spindle_b200.h.
It lets the CPU suite check the plan compiler (views, fusion, multi-output
merging, liveness packing, collective tables) against the oracle without a
GPU; the GPU tests then check the kernels themselves.
"""
from __future__ import annotations

import numpy as np

from paper_2401_11202_b200 import runtime as R


class Sim:
    def __init__(self, ex):
        self.ex = ex
        self.arena = np.full(ex.slice_elems * ex.ndev, np.nan, dtype=np.float32)
        self.tables = ex.table_blob
        self.arena[ex.zero_off:ex.zero_off + ex.zero_elems] = 0.0

    # addresses -> arena element index
    def idx(self, addr):
        return (int(addr) - self.ex.base) // 4

    def table(self, addr, dtype, n):
        o = int(addr) - self.ex.table_base
        return np.frombuffer(self.tables[o:o + n * np.dtype(dtype).itemsize].tobytes(), dtype=dtype)

    def dev_base(self, p):
        return p * self.ex.slice_elems

    def gather_view(self, p, off, strides, dims):
        dims = [int(d) for d in dims]
        index = np.full(dims, self.dev_base(p) + int(off), dtype=np.int64)
        for k, d in enumerate(dims):
            shape = [1] * len(dims)
            shape[k] = d
            index = index + np.arange(d, dtype=np.int64).reshape(shape) * int(strides[k])
        return self.arena[index]

    def eval_prog(self, x, ins):
        regs = {}
        for j, a in enumerate(ins):
            regs[j] = a
        with np.errstate(all="ignore"):
            for i in range(x.n_prog):
                ins_ = x.prog[i]
                op, a, b, imm = ins_.op, ins_.a, ins_.b, np.float32(x.imm[i])
                A = regs.get(a)
                B = regs.get(b)
                if op == R.OP["MOV"]:
                    v = A
                elif op == R.OP["ADD"]:
                    v = np.add(A, B)
                elif op == R.OP["MUL"]:
                    v = np.multiply(A, B)
                elif op == R.OP["NEG"]:
                    v = -A
                elif op == R.OP["EXP"]:
                    v = np.exp(A)
                elif op == R.OP["MAX"]:
                    v = np.maximum(A, B)
                elif op == R.OP["IMM"]:
                    v = imm
                elif op == R.OP["ADDI"]:
                    v = np.add(A, imm)
                elif op == R.OP["MULI"]:
                    v = np.multiply(A, imm)
                elif op == R.OP["IADD"]:
                    v = np.add(imm, A)
                elif op == R.OP["IMUL"]:
                    v = np.multiply(imm, A)
                else:
                    raise AssertionError(op)
                assert 0 <= ins_.dst < R.NREG
                regs[ins_.dst] = np.asarray(v, dtype=np.float32)
        return regs

    def run_ew(self, x: R.EwParams):
        dims = [x.dims[k] for k in range(x.rank)]
        for p in range(x.ndev):
            ins = [self.gather_view(p, x.inp[j].off, x.inp[j].stride, dims) for j in range(x.n_in)]
            regs = self.eval_prog(x, ins)
            for o in range(x.n_out):
                v = np.broadcast_to(regs[x.out_reg[o]], dims).reshape(-1)
                s = self.dev_base(p) + x.out_off[o]
                self.arena[s:s + v.size] = v

    def run_reduce(self, r: R.ReduceParams):
        x = r.x
        dims = [x.dims[k] for k in range(x.rank)]
        for p in range(x.ndev):
            ins = [self.gather_view(p, x.inp[j].off, x.inp[j].stride, dims) for j in range(x.n_in)]
            regs = self.eval_prog(x, ins)
            v = np.broadcast_to(regs[x.out_reg[0]], dims)
            axes = tuple(range(r.n_kept, x.rank))
            red = np.sum(v, axis=axes, dtype=np.float32) if r.monoid == 0 else np.max(v, axis=axes)
            red = np.asarray(red, dtype=np.float32).reshape(-1)
            s = self.dev_base(p) + r.out_off
            self.arena[s:s + red.size] = red

    # --- block-scaled 3xFP16 operands (gemm_h3.cu): pieces in the arena as fp16
    def run_split(self, q: R.SplitParams):
        h16 = self.arena.view(np.float16)
        for p in range(q.ndev):
            X = self.gather_view(p, q.src_off, (q.ld, 1), (q.rows, q.cols)).astype(np.float32)
            hi = np.zeros((q.rows, q.pitch), np.float16)
            lo = np.zeros((q.rows, q.pitch), np.float16)
            rb, cb = -(-q.rows // 128), -(-q.cols // 128)
            inv = np.zeros((rb, cb), np.float32)
            for i in range(rb):
                for j in range(cb):
                    blk = X[i * 128:(i + 1) * 128, j * 128:(j + 1) * 128]
                    m = np.float32(np.max(np.abs(blk)))
                    E = int((m.view(np.uint32) >> 23) & 0xFF)
                    e = 0 if (m == 0 or E == 255) else 141 - E
                    e = min(60, max(-60, e))
                    y = blk * np.float32(2.0 ** e)
                    h = y.astype(np.float16)
                    hi[i * 128:(i + 1) * 128, j * 128:j * 128 + blk.shape[1]] = h
                    lo[i * 128:(i + 1) * 128, j * 128:j * 128 + blk.shape[1]] = (y - h.astype(np.float32)).astype(np.float16)
                    inv[i, j] = np.float32(2.0 ** -e)
            d = 2 * (self.dev_base(p) + q.dst_off)
            n = q.rows * q.pitch
            h16[d:d + n] = hi.reshape(-1)
            h16[d + n:d + 2 * n] = lo.reshape(-1)
            s0 = self.dev_base(p) + q.scl_off
            self.arena[s0:s0 + inv.size] = inv.reshape(-1)

    def _h3_operand(self, p, off, scl, rows, cols):
        """fp32 view an h3 GEMM reads: (hi + lo) / s per block, from the arena."""
        h16 = self.arena.view(np.float16)
        pitch = (cols + 7) // 8 * 8
        d = 2 * (self.dev_base(p) + off)
        n = rows * pitch
        hi = h16[d:d + n].reshape(rows, pitch)[:, :cols].astype(np.float64)
        lo = h16[d + n:d + 2 * n].reshape(rows, pitch)[:, :cols].astype(np.float64)
        rb, cb = -(-rows // 128), -(-cols // 128)
        s0 = self.dev_base(p) + scl
        inv = self.arena[s0:s0 + rb * cb].reshape(rb, cb).astype(np.float64)
        f = np.repeat(np.repeat(inv, 128, axis=0), 128, axis=1)[:rows, :cols]
        return (hi + lo) * f

    def run_gemm(self, g: R.GemmParams):
        if g.h3_shared:
            for p in range(g.ndev):
                A = self._h3_operand(p, g.h3_a_off, g.h3_a_scl, *((g.K, g.M) if g.a_mn_major else (g.M, g.K)))
                B = self._h3_operand(p, g.h3_b_off, g.h3_b_scl, *((g.N, g.K) if g.b_k_major else (g.K, g.N)))
                C = (A.T if g.a_mn_major else A) @ (B.T if g.b_k_major else B)
                C = C.astype(np.float32)
                for m in range(g.M):
                    s = self.dev_base(p) + g.c_off + m * g.ldc
                    self.arena[s:s + g.N] = C[m]
            return
        for p in range(g.ndev):
            if g.a_mn_major:
                A = self.gather_view(p, g.a_off, (1, g.lda), (g.M, g.K))
            else:
                A = self.gather_view(p, g.a_off, (g.lda, 1), (g.M, g.K))
            if g.b_k_major:
                B = self.gather_view(p, g.b_off, (1, g.ldb), (g.K, g.N))
            else:
                B = self.gather_view(p, g.b_off, (g.ldb, 1), (g.K, g.N))
            S = max(1, g.splits) if g.sk_mode == 0 else 1     # sk_mode 1: reduced in the kernel
            for sp in range(S):
                k0, k1 = (g.K * sp) // S, (g.K * (sp + 1)) // S
                # partial k-ranges are whole 32-wide k-blocks in the kernel
                nk = -(-g.K // 32)
                k0, k1 = min(g.K, 32 * ((nk * sp) // S)), min(g.K, 32 * ((nk * (sp + 1)) // S))
                C = (A[:, k0:k1].astype(np.float64) @ B[k0:k1].astype(np.float64)).astype(np.float32)
                if g.epi != R.EPI_NONE:
                    self._epilogue(g, p, C)
                    continue
                for m in range(g.M):
                    s = self.dev_base(p) + g.c_off + (sp * g.M + m) * g.ldc
                    self.arena[s:s + g.N] = C[m]

    def _epilogue(self, g, p, C):
        """The fused GEMM epilogues (spindle_b200.h spx_epilogue), float32 ops."""
        f32 = np.float32
        X = [self.gather_view(p, g.epi_in_off[j], (g.epi_in_ld[j], 1), (g.M, g.N)) for j in range(2)
             if g.epi_in_ld[j] > 0]
        k0, k1 = f32(g.epi_imm[0]), f32(g.epi_imm[1])
        with np.errstate(all="ignore"):
            if g.epi == R.EPI_ADD:
                Y = [X[0] + C]
            elif g.epi == R.EPI_SQUARE:
                Y = [C, C * C]
            elif g.epi == R.EPI_MULSCALE:
                Y = [C * (X[0] * k0)]
            elif g.epi == R.EPI_MOMENTUM:
                m = X[0] * k0 + C
                Y = [m, X[1] + -(m * k1)]
            else:
                raise AssertionError(g.epi)
        for j, y in enumerate(Y):
            y = np.asarray(y, dtype=np.float32)
            for r in range(g.M):
                s = self.dev_base(p) + g.epi_out_off[j] + r * g.epi_out_ld[j]
                self.arena[s:s + g.N] = y[r]

    def run_gather(self, g: R.GatherParams):
        dims = [g.dims[k] for k in range(g.rank)]
        n = g.ndev * g.n_combo
        table = self.table(g.src_table, np.uint64, n)
        base = self.table(g.base_off, np.int64, g.ndev)
        dst = self.table(g.dst, np.uint64, g.ndev)
        l = np.indices(dims).reshape(len(dims), -1) if dims else np.zeros((0, 1), np.int64)
        for p in range(g.ndev):
            combo = np.zeros(l.shape[1], np.int64)
            soff = np.full(l.shape[1], base[p], np.int64)
            for k in range(g.rank):
                q, r = l[k] // g.ext[k], l[k] % g.ext[k]
                combo += q * g.cmul[k]
                soff += r * g.sstride[k]
            src = np.array([self.idx(table[p * g.n_combo + c]) for c in combo], dtype=np.int64)
            vals = self.arena[src + soff]
            d0 = self.idx(dst[p])
            self.arena[d0:d0 + vals.size] = vals

    def run_creduce(self, r: R.CreduceParams):
        dims = [r.dims[k] for k in range(r.rank)]
        mem = self.table(r.members, np.int32, r.ndev * r.n_members)
        src = self.table(r.src, np.uint64, max(r.ndev, int(mem.max()) + 1))
        base = self.table(r.base_off, np.int64, r.ndev)
        dst = self.table(r.dst, np.uint64, r.ndev)
        l = np.indices(dims).reshape(len(dims), -1) if dims else np.zeros((0, 1), np.int64)
        out = []
        for p in range(r.ndev):
            soff = np.full(l.shape[1], base[p], np.int64)
            for k in range(r.rank):
                soff += l[k] * r.sstride[k]
            acc = None
            for j in range(r.n_members):
                v = self.arena[self.idx(src[mem[p * r.n_members + j]]) + soff]
                acc = v if acc is None else (np.add(acc, v) if r.monoid == 0 else np.maximum(acc, v))
            out.append(acc)
        for p in range(r.ndev):          # all reads before writes (distinct buffers anyway)
            d0 = self.idx(dst[p])
            self.arena[d0:d0 + out[p].size] = out[p]

    def run(self):
        for kind, p in self.ex.records():
            {R.K_EW: self.run_ew, R.K_REDUCE: self.run_reduce, R.K_GEMM: self.run_gemm,
             R.K_GATHER: self.run_gather, R.K_CREDUCE: self.run_creduce, R.K_SPLIT: self.run_split}[kind](p)

    def upload(self, per_device):
        for p in range(self.ex.ndev):
            for a in self.ex.comp.arg_bufs:
                v = np.asarray(per_device[p][a], dtype=np.float32).reshape(-1)
                s = self.dev_base(p) + self.ex.off[a]
                self.arena[s:s + v.size] = v

    def results(self):
        f = self.ex.comp.f
        out = []
        for j, b in enumerate(self.ex.comp.result_bufs):
            dims = tuple(f.result_types[j].dims)
            n = int(np.prod(dims)) if dims else 1
            per = []
            for p in range(self.ex.ndev):
                s = self.dev_base(p) + self.ex.off[b]
                per.append(self.arena[s:s + n].reshape(dims).copy())
            out.append(per)
        return out


def sim_spmd(module, spec, inputs, tol=1e-5):
    """spmd_interpret through the record simulator (mirrors evaluator.spmd_interpret)."""
    from paper_2401_11202_b200.evaluator import _chunk_slices, unshard
    from paper_2401_11202_b200.executable import Executable
    f = module.func("main")
    mesh = module.mesh
    coords = mesh.coords()
    arrays = [np.asarray(inputs[n]) for n in f.arg_names()]
    per = []
    for c in coords:
        per.append({n: a[_chunk_slices(a.shape, spec.args[n], mesh, c)] for a, (n, _) in zip(arrays, f.args)})
    ex = Executable(module, dry=True)
    sim = Sim(ex)
    sim.upload(per)
    sim.run()
    res = sim.results()
    return [unshard(res[j], spec.results[j], mesh, coords, tol, f"result {j}") for j in range(len(res))], ex


def sim_dense(module, inputs):
    from paper_2401_11202_b200.evaluator import _Dense
    from paper_2401_11202_b200.executable import Executable
    f = module.func("main")
    ex = Executable(_Dense(module), devices=[0], dry=True)
    sim = Sim(ex)
    sim.upload([{n: np.asarray(inputs[n]) for n in f.arg_names()}])
    sim.run()
    return [r[0] for r in sim.results()], ex


PEER_SHIFT = 36


def _peer_of(addr):
    """(member rank or -1 for the own arena, address in that member's arena):
    dry peer mappings sit at DRY_BASE + (rank + 1) << PEER_SHIFT."""
    from paper_2401_11202_b200.executable import Executable
    tag = (int(addr) - Executable.DRY_BASE) >> PEER_SHIFT
    return (tag - 1 if tag > 0 else -1), int(addr) - (tag << PEER_SHIFT)


def _dry_comms(ex, peer):
    if peer:
        # every dry arena has base DRY_BASE; a peer's arena is "mapped" at
        # DRY_BASE + (rank + 1) << PEER_SHIFT, so an address names its member
        me = ex.comp.devices[0]
        ex.peer_bases = [ex.base if r == me else ex.base + ((r + 1) << PEER_SHIFT)
                         for r in range(ex.comp.mesh.device_count)]
    return {k: i for i, k in enumerate(ex.comm_keys())}


def sim_nccl(module, spec, inputs, tol=1e-5, peer=False):
    """The one-process-per-GPU (NCCL) lowering, simulated: one dry Executable
    per rank, records executed in lockstep, NCCL records combined across the
    ranks of each communicator group (rank order = group order)."""
    from paper_2401_11202_b200.evaluator import _chunk_slices, unshard
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.session import comm_plan
    f = module.func("main")
    mesh = module.mesh
    coords = mesh.coords()
    world = len(coords)
    exs, sims = [], []
    probe = Executable(module, devices=[0], comm_mode="nccl", dry=True,
                       comm_factory=lambda ex: _dry_comms(ex, False))
    plan = comm_plan(probe)
    for r in range(world):
        ex = Executable(module, devices=[r], comm_mode="nccl", dry=True,
                        comm_factory=lambda ex: _dry_comms(ex, peer))
        exs.append(ex)
        s = Sim(ex)
        a = {n: np.asarray(inputs[n])[_chunk_slices(np.shape(inputs[n]), spec.args[n], mesh, coords[r])]
             for n in f.arg_names()}
        s.upload([a])
        sims.append(s)
    nrec = len(exs[0].records())
    assert all(len(e.records()) == nrec for e in exs)
    for i in range(nrec):
        kind = exs[0].records()[i][0]
        if kind == R.K_PEER and exs[0].records()[i][1].kind == 3:
            continue                     # barrier only (copy-engine reduce-scatter handshakes)
        if kind == R.K_PEER:
            # each member reads every member's source (same arena offset) and
            # folds in member order; all reads happen before any write
            outs = []
            for r in range(world):
                p = exs[r].records()[i][1]
                grp = plan[[k for k, _ in plan].index(exs[r].peer_slots()[p.slot][0])][1]
                grp = next(g for g in grp if r in g)
                assert grp.index(r) == p.me and len(grp) == p.n
                acc = None
                for j, m in enumerate(grp):
                    o = sims[m].idx(_peer_of(p.src[j])[1])
                    x = sims[m].arena[o:o + p.count]
                    if p.kind == 1:          # all-gather: member chunks in member order
                        acc = x.copy() if acc is None else np.concatenate([acc, x])
                        continue
                    acc = x.copy() if acc is None else (np.add(acc, x) if p.monoid == 0 else np.maximum(acc, x))
                outs.append((r, sims[r].idx(p.dst), acc))
            for r, d0, acc in outs:
                sims[r].arena[d0:d0 + acc.size] = acc
            continue
        if kind == R.K_COPY:
            # device-to-device copies (copy-engine all-gather): read every source first
            outs = []
            for r in range(world):
                p = exs[r].records()[i][1]
                assert p.dir == 2
                m, a = _peer_of(p.host)
                m = r if m < 0 else m
                o = sims[m].idx(a)
                outs.append((r, sims[r].idx(p.dev), sims[m].arena[o:o + p.bytes // 4].copy()))
            for r, d0, x in outs:
                sims[r].arena[d0:d0 + x.size] = x
            continue
        if kind != R.K_NCCL:
            for s, e in zip(sims, exs):
                k, p = e.records()[i]
                {R.K_EW: s.run_ew, R.K_REDUCE: s.run_reduce, R.K_GEMM: s.run_gemm,
                 R.K_GATHER: s.run_gather, R.K_CREDUCE: s.run_creduce, R.K_SPLIT: s.run_split}[k](p)
            continue
        p0 = exs[0].records()[i][1]
        key, groups = plan[p0.comm]
        for grp in groups:
            ps = [exs[r].records()[i][1] for r in grp]
            cnt = ps[0].count
            sends = [sims[r].arena[sims[r].idx(p.send):sims[r].idx(p.send) + (cnt * len(grp)
                     if p.kind in (R.NCCL_REDUCESCATTER, R.NCCL_ALLTOALL) else cnt)].copy()
                     for r, p in zip(grp, ps)]
            outs = []
            if p0.kind == R.NCCL_ALLREDUCE:
                acc = sends[0]
                for x in sends[1:]:
                    acc = np.add(acc, x) if p0.monoid == 0 else np.maximum(acc, x)
                outs = [acc] * len(grp)
            elif p0.kind == R.NCCL_ALLGATHER:
                outs = [np.concatenate(sends)] * len(grp)
            elif p0.kind == R.NCCL_REDUCESCATTER:
                acc = sends[0]
                for x in sends[1:]:
                    acc = np.add(acc, x) if p0.monoid == 0 else np.maximum(acc, x)
                outs = [acc[j * cnt:(j + 1) * cnt] for j in range(len(grp))]
            else:  # all-to-all: rank j receives piece j of every sender, in sender order
                outs = [np.concatenate([sends[s][j * cnt:(j + 1) * cnt] for s in range(len(grp))])
                        for j in range(len(grp))]
            for r, p, o in zip(grp, ps, outs):
                d0 = sims[r].idx(p.recv)
                sims[r].arena[d0:d0 + o.size] = o
    res = [s.results() for s in sims]           # [rank][result][device0]
    out = []
    for j in range(len(f.results)):
        out.append(unshard([res[r][j][0] for r in range(world)], spec.results[j], mesh, coords, tol, f"result {j}"))
    return out, exs
