"""Resident sessions: compile once, keep inputs in HBM, step many times.

`Session` is the API the benchmark and long-running users call (the drop-in
`spmd_interpret` is one-shot: shard, upload, run, download, unshard).  Two
hosting modes (see executable.py):

  Session(module, sharding)                      all mesh devices on this GPU
  Session(module, sharding, mode="nccl")         one mesh device per process;
      rank/world/local_rank from torch.distributed (torchrun), NCCL
      communicators per mesh-axis group created through ncclCommInitRank with
      unique ids broadcast over torch.distributed (`make_nccl_comms`).
"""
from __future__ import annotations

import numpy as np

from . import runtime as R
from .evaluator import _Dense, _chunk_slices, unshard
from .executable import Executable


def nccl_uid() -> bytes:
    lib = R.load()
    buf = (R.C.c_uint8 * 128)()
    R.call(lib.spx_nccl_get_unique_id, R.C.cast(buf, R.C.c_void_p))
    return bytes(buf)


def nccl_comm_init(uid: bytes, nranks: int, rank: int) -> int:
    lib = R.load()
    buf = (R.C.c_uint8 * 128).from_buffer_copy(uid)
    out = R.C.c_int()
    R.call(lib.spx_comm_init, R.C.cast(buf, R.C.c_void_p), nranks, rank, R.C.byref(out))
    return out.value


def ipc_handle(ptr: int) -> bytes:
    lib = R.load()
    buf = (R.C.c_uint8 * 64)()
    R.call(lib.spx_ipc_get_handle, ptr, R.C.cast(buf, R.C.c_void_p))
    return bytes(buf)


def ipc_open(handle: bytes) -> int:
    lib = R.load()
    buf = (R.C.c_uint8 * 64).from_buffer_copy(handle)
    out = R.C.c_uint64()
    R.call(lib.spx_ipc_open, R.C.cast(buf, R.C.c_void_p), R.C.byref(out))
    return out.value


def map_peer_arenas(ex: Executable, rank: int, allgather):
    """Exchange CUDA IPC handles of every rank's arena (`allgather(obj) ->
    [obj per rank]`) and map the peers' arenas into this process; enables the
    peer-memory all-reduce records (csrc/peer.cu).  The arena's flag words are
    zeroed (and synchronised) before any handle is published."""
    ex.device.sync()
    handles = allgather(ipc_handle(ex.base))
    bases = []
    for r, h in enumerate(handles):
        if r == rank:
            bases.append(ex.base)
        else:
            ptr = ipc_open(h)
            ex._peer_handles.append(ptr)
            bases.append(ptr)
    ex.peer_bases = bases


def comm_plan(ex: Executable):
    """[(axes key, groups)] in the shared deterministic order."""
    c = ex.comp
    return [(key, c._groups(list(key))) for key in ex.comm_keys()]


def make_nccl_comms(ex: Executable, rank: int, broadcast, get_uid=nccl_uid, init=nccl_comm_init,
                    allgather=None):
    """One communicator per axes key; NCCL rank = position in the group's
    device order (the reference's group order, spmd_interp.py:57-63).
    `broadcast(obj) -> obj` shares rank 0's unique ids with every rank;
    with `allgather`, the peers' arenas are also mapped (map_peer_arenas)."""
    plan = comm_plan(ex)
    if allgather is not None and ex.wants_peer and plan:
        map_peer_arenas(ex, rank, allgather)
    import os
    if os.environ.get("SPX_NCCL_NONE", "0") == "1":
        # peer-memory collectives only (every collective of the program must take
        # the peer path; an NCCL record then fails loudly): lets tools/nccl_parity.py
        # run 8 ranks on a 4-GPU box, two processes per GPU, where NCCL refuses
        # duplicate devices
        return {key: -1 for key, _ in plan}
    uids = None
    if rank == 0:
        uids = {(key, gi): get_uid() for key, groups in plan for gi in range(len(groups))}
    uids = broadcast(uids)
    comms = {}
    for key, groups in plan:
        gi = next(i for i, g in enumerate(groups) if rank in g)
        grp = groups[gi]
        comms[key] = init(uids[(key, gi)], len(grp), grp.index(rank))
    return comms


def torch_allgather(obj):
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def torch_broadcast(obj):
    import torch.distributed as dist
    box = [obj]
    dist.broadcast_object_list(box, src=0)
    return box[0]


class Session:
    def __init__(self, module, sharding=None, *, mode="local", device: R.Device | None = None,
                 rank: int = 0, world: int = 1, local_rank: int = 0, gemm_path: int = 0,
                 func: str = "main", broadcast=torch_broadcast, allgather=torch_allgather, io: bool = False):
        """io=True: the plan also copies every argument in and every result out
        (copy records overlapped with the step) -- use `call` / `call_local`, not
        `step`, which would replay the copies with stale host buffers."""
        self.module = module
        self.sharding = sharding
        self.mode = mode
        self.func = module.func(func)
        if sharding is None or module.mesh is None:
            target = _Dense(module) if module.mesh is not None else module
            self.mesh = None
            self.coords = [{}]
            self.device = device or R.Device(local_rank)
            self.ex = Executable(target, func, device=self.device, devices=[0], gemm_path=gemm_path, io=io)
            self.hosted = [0]
        elif mode == "local":
            self.mesh = module.mesh
            self.coords = self.mesh.coords()
            self.device = device or R.Device(local_rank)
            self.ex = Executable(module, func, device=self.device, gemm_path=gemm_path, io=io)
            self.hosted = list(range(len(self.coords)))
        else:
            self.mesh = module.mesh
            self.coords = self.mesh.coords()
            if self.mesh.device_count != world:
                raise ValueError(f"mesh has {self.mesh.device_count} devices, world size is {world}")
            self.device = device or R.Device(local_rank)
            self.ex = Executable(module, func, device=self.device, devices=[rank], comm_mode="nccl",
                                 gemm_path=gemm_path, io=io,
                                 comm_factory=lambda ex: make_nccl_comms(ex, rank, broadcast,
                                                                         allgather=allgather))
            self.hosted = [rank]
        self.rank = rank

    # -- inputs -----------------------------------------------------------
    def local_inputs(self, global_inputs: dict) -> list[dict]:
        f = self.func
        out = []
        for d in self.hosted:
            env = {}
            for n, t in f.args:
                a = np.asarray(global_inputs[n], dtype=np.float32)
                if self.mesh is not None:
                    a = a[_chunk_slices(a.shape, self.sharding.args[n], self.mesh, self.coords[d])]
                if tuple(a.shape) != tuple(t.dims):
                    raise ValueError(f"arg %{n}: sharded input is {a.shape}, local signature wants {t.dims}")
                env[n] = a
            out.append(env)
        return out

    def load(self, global_inputs: dict):
        self.ex.upload_args(self.local_inputs(global_inputs))
        self.device.sync()
        self._rank_barrier()      # peers may gather these arguments by copy engine (no device handshake)

    def _rank_barrier(self):
        if self.mode == "nccl":
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                dist.barrier()

    def arg_addr(self, name: str, p: int = 0) -> int:
        return self.ex.addr(p, name)

    # -- execution --------------------------------------------------------
    def run(self):
        self.ex.plan.run()

    def capture(self):
        self.ex.plan.capture()

    # -- input pipeline -----------------------------------------------------
    def feed(self, host: dict):
        """Stage the NEXT step's inputs: `host[name]` are pinned host arrays of
        local (already sharded) args; they go host->device on a copy stream
        into one of two staging slots, overlapping the step that is running.
        The next `step()` waits for the copy, moves the slot into the arg
        buffers (device-to-device) and runs.  Hosted device 0 (nccl mode:
        this rank's device).  In nccl mode only feed arguments no other rank
        gathers by copy engine (the sharded batch -- ZeRO-3 gathers parameters),
        or set SPX_CE_AG=0: a step's argument update has no cross-rank handshake."""
        dev = self.device
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = dev.new_stream()
            self._stage = {}
            self._ready = [dev.event(), dev.event()]
            self._consumed = [dev.event(), dev.event()]
            self._fed = 0
            self._pending = []
        slot = self._fed % 2
        if self._fed >= 2:
            # the slot's previous batch must have been moved into the args
            dev.wait(self._consumed[slot], self._copy_stream)
        for nm, arr in host.items():
            if nm not in self._stage:
                self._stage[nm] = (dev.malloc(arr.nbytes), dev.malloc(arr.nbytes), arr.nbytes)
            dev.h2d_async(self._stage[nm][slot], arr, self._copy_stream)
        dev.record(self._ready[slot], self._copy_stream)
        self._pending.append((slot, list(host)))
        self._fed += 1

    def step(self):
        if getattr(self, "_pending", None):
            slot, names = self._pending.pop(0)
            dev = self.device
            dev.wait(self._ready[slot])
            for nm in names:
                dev.d2d(self.arg_addr(nm), self._stage[nm][slot], self._stage[nm][2])
            dev.record(self._consumed[slot])
        self.ex.plan.replay()

    def sync(self):
        if self.mode == "nccl":
            self.device.sync_watch()      # NCCL async errors / peer timeouts raise instead of hanging
        else:
            self.device.sync()

    def launch_count(self) -> int:
        return self.ex.plan.launch_count()

    def results(self):
        return self.ex.download_results()

    def call(self, global_inputs: dict):
        """One step with every input coming from host memory and every result
        going back to it -- the drop-in call's data movement (spmd_interpret:
        shard, copy in, run, copy out) for this process's mesh devices:
        returns [result j][hosted device] local arrays."""
        return self.call_local(self.local_inputs(global_inputs))

    def call_local(self, local_inputs: list[dict]):
        """`call` with inputs already sharded: local_inputs[hosted device][arg].
        One process per GPU: the ranks first meet at a barrier, since a peer may
        still be reading this rank's arguments (copy-engine all-gathers of the
        ZeRO-3 parameters) for the previous call."""
        self._rank_barrier()
        if self.ex.io:
            res = self.ex.call(local_inputs, replay=self.ex.plan.captured)
            if not self.ex.plan.captured:
                self.ex.plan.capture()
            return res
        self.ex.upload_args(local_inputs)
        if self.ex.plan.captured:
            self.ex.plan.replay()
        else:
            self.ex.plan.run()
        return self.ex.download_results()

    def result_addr(self, j: int, p: int = 0) -> int:
        return self.ex.addr(p, self.ex.comp.result_bufs[j])

    def global_results(self, tol=1e-5):
        res = self.results()
        if self.mesh is None:
            return [r[0] for r in res]
        return [unshard(res[j], self.sharding.results[j], self.mesh, self.coords, tol, f"result {j}")
                for j in range(len(res))]

    def close(self):
        self.ex.close()
