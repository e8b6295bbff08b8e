"""Shared test helpers.

GPU tests are marked `@pytest.mark.gpu`; the CPU suite (`-m "not gpu"`) covers
the oracle against the reference's golden vectors, the host-side plan
compiler, the multi-process (gloo) host logic, and that the C-ABI library
loads and exports every declared symbol.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# the reference package (tactic front end) where it exists: this container's
# source tree, or the offline install that travels to the GPU box
# (DESIGN.md §6); appended before the backend is imported so the backend's
# errors subclass the reference's
for _ref in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(_ref) and _ref not in sys.path:
        sys.path.append(_ref)

GOLDEN = os.path.join(ROOT, "tests", "golden")
TOL = 1e-5


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


_CASES = None
_OUTS = None


def golden_cases():
    global _CASES
    if _CASES is None:
        with open(os.path.join(GOLDEN, "cases.json")) as fh:
            _CASES = json.load(fh)
    return _CASES


def golden_outputs():
    global _OUTS
    if _OUTS is None:
        _OUTS = dict(np.load(os.path.join(GOLDEN, "outputs.npz")))
    return _OUTS


def case_inputs(case, module, seed):
    """Rebuild a case's inputs from its recipe (tests/golden/make_golden.py)."""
    from oracle.spmd_oracle import random_inputs
    r = case["inputs"]
    f = module.func("main")
    if r["kind"] == "random_inputs":
        return random_inputs(module, seed=seed, scale=r["scale"])
    if r["kind"] == "normal":
        rng = np.random.default_rng(r["seed"])
        return {n: rng.standard_normal(t.dims).astype(np.float32) for n, t in f.args}
    if r["kind"] == "ones":
        return {n: np.ones(t.dims, np.float32) for n, t in f.args}
    if r["kind"] == "arange":
        return {n: np.arange(float(np.prod(t.dims)), dtype=np.float32).reshape(t.dims)
                for n, t in f.args}
    raise ValueError(r)


def case_expected(case, seed, which):
    outs = golden_outputs()
    return [outs[f"{case['key']}/s{seed}/{which}/{j}"] for j in range(case["n_out"])]


requires_gpu = pytest.mark.skipif(not gpu_available(), reason="no CUDA device")
