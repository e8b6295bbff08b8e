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

import threading

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


def _check_dtype(arrays):
    for a in arrays:
        if a.dtype != np.float32:
            if a.dtype.kind == "f":
                continue    # computed in f32 (the backend's arithmetic type)
            raise TypeError(f"backend computes f32; got {a.dtype}")


def spmd_interpret(module, sharding, inputs, func: str = "main", tol: float = 1e-5,
                   device: R.Device | None = None, gemm_path: int = 0) -> list[np.ndarray]:
    """Run a localized module on global inputs on the B200; returns global outputs."""
    f = module.func(func)
    mesh = module.mesh
    if mesh is None:
        raise ValueError("spmd execution requires a mesh")
    coords = mesh.coords()
    arrays = _arrays(f, inputs)
    _check_dtype(arrays)
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
        ex = Executable(module, func, device=dev, gemm_path=gemm_path)
        try:
            ex.upload_args(per_device)
            ex.run()
            res = ex.download_results()
        finally:
            ex.close()
    out = []
    for j, r in enumerate(f.results):
        out.append(unshard(res[j], sharding.results[j], mesh, coords, tol, f"result {j} (%{r})"))
    return out


def interpret(module, inputs, func: str = "main", device: R.Device | None = None,
              gemm_path: int = 0) -> list[np.ndarray]:
    """Dense (single-device) execution on the B200 (interp.py:117-132 semantics)."""
    f = module.func(func)
    arrays = _arrays(f, inputs)
    if len(arrays) != len(f.args):
        raise EvalError(f"@{f.name} takes {len(f.args)} args, got {len(arrays)}")
    for a, (n, t) in zip(arrays, f.args):
        if tuple(a.shape) != tuple(t.dims):
            raise EvalError(f"arg %{n} expects shape {tuple(t.dims)}, got {tuple(a.shape)}")
    _check_dtype(arrays)
    if any(op.kind in ("all_slice", "all_gather", "all_reduce", "reduce_scatter", "all_to_all")
           for op in f.ops):
        raise EvalError("collective ops have no dense semantics; use spmd_interpret")
    dense = _Dense(module)
    with _LOCK:
        dev = device or default_device()
        try:
            ex = Executable(dense, func, device=dev, devices=[0], gemm_path=gemm_path)
        except UnsupportedProgram as e:
            raise EvalError(str(e)) from e
        try:
            ex.upload_args([{n: a for a, (n, _) in zip(arrays, f.args)}])
            ex.run()
            res = ex.download_results()
        finally:
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
