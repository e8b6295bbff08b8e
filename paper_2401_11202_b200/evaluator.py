"""Drop-in B200 evaluator with the reference's interface.

`spmd_interpret` mirrors /root/reference/pkg/src/spindle/spmd_interp.py:157-197
(same signature, argument meaning, return type and exceptions): inputs are
GLOBAL arrays sharded by the callee per the ShardingSpec, every mesh device's
local program runs on the B200 (all devices co-located on one GPU, collectives
as in-GPU group kernels), and outputs are reassembled with the same replica
consensus check (`unshard`, :138-154) raising `DivergenceError`.

`interpret` mirrors interp.py:117-132 for straight-line (dense / 1-device)
modules: the single-GPU data point of the benchmark.
"""
from __future__ import annotations

import hashlib
import json
import os
import threading
from collections import OrderedDict

import numpy as np

from . import runtime as R
from .executable import Executable
from .plan import UnsupportedProgram


try:  # when the reference package is importable, our errors ARE its errors too
    from spindle.spmd_interp import DivergenceError as _RefDivergence  # type: ignore
    from spindle.interp import EvalError as _RefEvalError  # type: ignore
except Exception:  # pragma: no cover - the GPU box has no reference
    _RefDivergence = Exception
    _RefEvalError = Exception


class DivergenceError(_RefDivergence):
    """Device replicas disagree on a value that must be replicated (spmd_interp.py:21-22)."""


class EvalError(_RefEvalError):
    """interp.py:16-17"""


def relative_error(got, want) -> float:
    """spmd_interp.py:25-31"""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.shape != want.shape:
        return float("inf")
    denom = float(np.max(np.abs(want))) + 1e-12
    return float(np.max(np.abs(got - want))) / denom


_DEVICE = None
_LOCK = threading.Lock()


def default_device() -> R.Device:
    global _DEVICE
    if _DEVICE is None:
        _DEVICE = R.Device(0)
    return _DEVICE


def _chunk_index(coord, axes, mesh):
    idx = 0
    for ax in axes:
        idx = idx * mesh.size(ax) + coord[ax]
    return idx


def _chunk_slices(gdims, apd, mesh, coord):
    out = []
    for d, axes in enumerate(apd):
        n = 1
        for ax in axes:
            n *= mesh.size(ax)
        ext = gdims[d] // n
        i = _chunk_index(coord, axes, mesh)
        out.append(slice(i * ext, (i + 1) * ext))
    return tuple(out)


def _global_dims(local_dims, apd, mesh):
    out = list(local_dims)
    for d, axes in enumerate(apd):
        for ax in axes:
            out[d] *= mesh.size(ax)
    return tuple(out)


def unshard(locals_by_device, apd, mesh, coords, tol, label):
    """Reassemble a global result; replicas of a chunk must agree within tol."""
    gdims = _global_dims(locals_by_device[0].shape, apd, mesh)
    out = np.zeros(gdims, dtype=locals_by_device[0].dtype)
    seen = {}
    for i, c in enumerate(coords):
        key = tuple(_chunk_index(c, axes, mesh) for axes in apd)
        sl = _chunk_slices(gdims, apd, mesh, c)
        if key in seen:
            err = relative_error(locals_by_device[i], out[sl])
            if err > tol:
                raise DivergenceError(
                    f"{label}: replicas disagree (relative error {err:.3e} > {tol:.1e}) "
                    f"between device {seen[key]} and device {i}")
        else:
            seen[key] = i
            out[sl] = locals_by_device[i]
    return out


def _arrays(f, inputs):
    if isinstance(inputs, dict):
        return [np.asarray(inputs[n]) for n in f.arg_names()]
    return [np.asarray(a) for a in inputs]


def _cdtype(arrays):
    """The reference computes in `np.result_type` of the inputs
    (spmd_interp.py:173, interp.py:127; constants adopt it, interp.py:39-41).
    The backend's arithmetic types are f32 and i32 (the IR's element kinds,
    ir.py:14); any other result type -- f64 inputs, or f32 mixed with i32,
    which numpy promotes to f64 -- is refused rather than silently computed
    in another precision."""
    cdtype = np.result_type(*[a.dtype for a in arrays]) if arrays else np.dtype(np.float32)
    if cdtype not in (np.dtype(np.float32), np.dtype(np.int32)):
        raise TypeError(f"the B200 backend computes in float32 or int32; these inputs compute in "
                        f"{cdtype} (np.result_type of {sorted({str(a.dtype) for a in arrays})})")
    return cdtype


# ---------------------------------------------------------------------------
# compiled-plan cache: one Executable -- plan records, arena,
# TMA descriptors, CUDA graph -- per (module, ShardingSpec, func, knobs),
# keyed by a fingerprint of the IR, so repeated calls of the drop-in only
# copy inputs in, replay the step and copy results out.
# ---------------------------------------------------------------------------

def _jsonable(x):
    if isinstance(x, dict):
        return {str(k): _jsonable(v) for k, v in sorted(x.items(), key=lambda kv: str(kv[0]))}
    if isinstance(x, (list, tuple)):
        return [_jsonable(v) for v in x]
    if isinstance(x, (str, int, float, bool)) or x is None:
        return x
    if hasattr(x, "dims"):
        return {"dims": list(x.dims), "elem": getattr(x, "elem", "f32")}
    return str(x)


def fingerprint(module, func="main") -> str:
    """sha256 over the function's signature, ops (kind, names, types, attrs)
    and the mesh; works on this package's IR objects and on the reference's."""
    h = hashlib.sha256()
    mesh = getattr(module, "mesh", None)
    h.update(repr(None if mesh is None else [(n, mesh.size(n)) for n in mesh.names()]).encode())
    f = module.func(func)
    h.update(json.dumps([[n, list(t.dims), getattr(t, "elem", "f32")] for n, t in f.args]).encode())
    for op in f.ops:
        h.update(json.dumps([op.kind, list(op.results), list(op.operands),
                             [[list(t.dims), getattr(t, "elem", "f32")] for t in op.result_types],
                             _jsonable(op.attrs)]).encode())
        if getattr(op, "regions", None):
            raise EvalError(f"op {op.kind!r} carries regions: localize the module first")
    h.update(json.dumps(list(f.results)).encode())
    return h.hexdigest()


class PlanCache:
    """LRU of compiled Executables.  Bounded by entry count (SPX_PLAN_CACHE,
    default 4) and by arena bytes (SPX_PLAN_CACHE_BYTES, default 160 GiB of
    the B200's 180 GB: one C3-sized plan, 96 GB, must stay resident; a build
    that runs out of memory evicts everything and retries once);
    SPX_PLAN_CACHE=0 disables caching (every call builds and frees its plan)."""

    def __init__(self):
        self.entries: "OrderedDict[tuple, Executable]" = OrderedDict()
        self.hits = self.misses = 0

    @staticmethod
    def limits():
        return (int(os.environ.get("SPX_PLAN_CACHE", "4")),
                int(os.environ.get("SPX_PLAN_CACHE_BYTES", str(160 << 30))))

    def bytes(self) -> int:
        return sum(ex.dev_stride * ex.ndev for ex in self.entries.values())

    def get(self, key):
        ex = self.entries.get(key)
        if ex is not None:
            self.entries.move_to_end(key)
            self.hits += 1
        return ex

    def put(self, key, ex):
        self.misses += 1
        n_max, b_max = self.limits()
        if n_max <= 0:
            return False
        self.entries[key] = ex
        while self.entries and (len(self.entries) > n_max or self.bytes() > b_max):
            _, old = self.entries.popitem(last=False)
            if old is ex:
                return False
            old.close()
        return True

    def clear(self):
        while self.entries:
            _, ex = self.entries.popitem(last=False)
            ex.close()


_CACHE = PlanCache()


def plan_cache() -> PlanCache:
    return _CACHE


def _knobs():
    return tuple(sorted((k, v) for k, v in os.environ.items() if k.startswith("SPX_")))


def _make_room(dev):
    """before_alloc hook: evict cached plans (LRU) until the new arena fits in
    the device's free memory with a margin for launches and workspaces."""
    margin = int(os.environ.get("SPX_PLAN_MARGIN_BYTES", str(6 << 30)))

    def hook(nbytes):
        while _CACHE.entries and dev.mem_info()[0] < nbytes + margin:
            _, old = _CACHE.entries.popitem(last=False)
            old.close()
    return hook


def _build(key, make):
    """Executable for `key` from the cache, or built by make() and cached."""
    ex = _CACHE.get(key)
    if ex is not None:
        return ex, True
    try:
        ex = make()
    except R.BackendError as e:
        if "out of memory" not in str(e) or not _CACHE.entries:
            raise
        _CACHE.clear()           # cached arenas hold the memory: drop them and retry once
        ex = make()
    return ex, _CACHE.put(key, ex)


def _io() -> bool:
    """Copies inside the plan, overlapped with the step (Executable io=True);
    SPX_IO_OVERLAP=0: copy in, run, copy out."""
    return os.environ.get("SPX_IO_OVERLAP", "1") != "0"


def _check_range():
    """The block-scaled fp16 splits clamp a block's scale to 2^+-60; a block whose
    maximum lies outside [2^-45, 2^75] keeps only ~2^-40-of-its-maximum accuracy
    for its small elements.  Report it (warning, or RangeError-like
    FloatingPointError with SPX_STRICT_RANGE=1) instead of degrading silently."""
    n = R.h3_range_events(reset=True)
    if n:
        msg = (f"{n} operand block(s) of the block-scaled fp16 GEMM split had a maximum outside "
               f"[2^-45, 2^75]; their small elements lose precision (set SPX_GEMM_H3=0 for the 3xTF32 path)")
        if os.environ.get("SPX_STRICT_RANGE", "0") == "1":
            raise FloatingPointError(msg)
        import warnings
        warnings.warn(msg, RuntimeWarning, stacklevel=3)


def _execute(ex, per_device, cached):
    res = _execute_plan(ex, per_device, cached)
    _check_range()
    return res


def _execute_plan(ex, per_device, cached):
    if ex.io:
        res = ex.call(per_device, replay=cached and ex.plan.captured)
        if cached and not ex.plan.captured:
            ex.plan.capture()    # later calls replay the step, copies included, as one CUDA graph
        return res
    ex.upload_args(per_device)
    if cached and ex.plan.captured:
        ex.plan.replay()
    else:
        ex.run()
        if cached:
            ex.plan.capture()    # later calls replay the whole step as one CUDA graph
    return ex.download_results()


def last_executable():
    """The Executable of the most recent drop-in call (tests inspect its
    records to check which kernels ran)."""
    return _LAST


_LAST = None


def spmd_interpret(module, sharding, inputs, func: str = "main", tol: float = 1e-5,
                   device: R.Device | None = None, gemm_path: int = 0) -> list[np.ndarray]:
    """Run a localized module on global inputs on the B200; returns global outputs."""
    global _LAST
    f = module.func(func)
    mesh = module.mesh
    if mesh is None:
        raise ValueError("spmd execution requires a mesh")
    coords = mesh.coords()
    arrays = _arrays(f, inputs)
    cdtype = _cdtype(arrays)
    per_device = []
    for c in coords:
        env = {}
        for a, (n, t) in zip(arrays, f.args):
            local = a[_chunk_slices(a.shape, sharding.args[n], mesh, c)]
            if tuple(local.shape) != tuple(t.dims):
                raise ValueError(f"arg %{n}: sharded input is {tuple(local.shape)}, "
                                 f"local signature wants {tuple(t.dims)}")
            env[n] = local
        per_device.append(env)
    with _LOCK:
        dev = device or default_device()
        key = ("spmd", fingerprint(module, func), func, gemm_path, str(cdtype), dev.ordinal, _knobs())
        ex, cached = _build(key, lambda: Executable(module, func, device=dev, gemm_path=gemm_path,
                                                    dtype=cdtype, io=_io(), before_alloc=_make_room(dev)))
        _LAST = ex
        try:
            res = _execute(ex, per_device, cached)
        finally:
            if not cached:
                ex.close()
    out = []
    for j, r in enumerate(f.results):
        out.append(unshard(res[j], sharding.results[j], mesh, coords, tol, f"result {j} (%{r})"))
    return out


def interpret(module, inputs, func: str = "main", device: R.Device | None = None,
              gemm_path: int = 0) -> list[np.ndarray]:
    """Dense (single-device) execution on the B200 (interp.py:117-132 semantics)."""
    global _LAST
    f = module.func(func)
    arrays = _arrays(f, inputs)
    if len(arrays) != len(f.args):
        raise EvalError(f"@{f.name} takes {len(f.args)} args, got {len(arrays)}")
    for a, (n, t) in zip(arrays, f.args):
        if tuple(a.shape) != tuple(t.dims):
            raise EvalError(f"arg %{n} expects shape {tuple(t.dims)}, got {tuple(a.shape)}")
    cdtype = _cdtype(arrays)
    if any(op.kind in ("all_slice", "all_gather", "all_reduce", "reduce_scatter", "all_to_all")
           for op in f.ops):
        raise EvalError("collective ops have no dense semantics; use spmd_interpret")
    dense = _Dense(module)
    with _LOCK:
        dev = device or default_device()
        key = ("dense", fingerprint(dense, func), func, gemm_path, str(cdtype), dev.ordinal, _knobs())

        def make():
            try:
                return Executable(dense, func, device=dev, devices=[0], gemm_path=gemm_path, dtype=cdtype,
                                  io=_io(), before_alloc=_make_room(dev))
            except UnsupportedProgram as e:
                raise EvalError(str(e)) from e
        ex, cached = _build(key, make)
        _LAST = ex
        try:
            res = _execute(ex, [{n: a for a, (n, _) in zip(arrays, f.args)}], cached)
        finally:
            if not cached:
                ex.close()
    return [r[0] for r in res]


class _Dense:
    """A module viewed without its mesh (dense programs run as one device)."""

    def __init__(self, module):
        self.funcs = module.funcs
        self.mesh = None

    def func(self, name="main"):
        return self._m_func(name)

    def _m_func(self, name):
        for f in self.funcs:
            if f.name == name:
                return f
        raise KeyError(f"no function named {name!r}")
