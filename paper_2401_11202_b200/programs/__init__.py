"""Cached partitioned programs (tools/make_programs.py output).

Each directory holds the artefacts the reference CLI dumps (`cli.py:79-91`):
dense.ir (unpartitioned module), local.ir + sharding.json (localized SPMD
module and its ShardingSpec), meta.json (counts, simulator cost, params).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

from ..ir import ShardingSpec, parse_module

HERE = os.path.dirname(os.path.abspath(__file__))


@dataclass
class Program:
    name: str
    meta: dict
    dense_text: str
    local_text: str | None
    sharding_json: dict | None
    _dense = None
    _local = None

    @property
    def dense(self):
        if self._dense is None:
            self._dense = parse_module(self.dense_text)
        return self._dense

    @property
    def local(self):
        if self._local is None and self.local_text is not None:
            self._local = parse_module(self.local_text)
        return self._local

    @property
    def sharding(self):
        return ShardingSpec.from_json(self.sharding_json) if self.sharding_json else None

    @property
    def batch(self) -> int:
        return int(self.meta["params"]["batch"])


def list_programs():
    return sorted(d for d in os.listdir(HERE) if os.path.isdir(os.path.join(HERE, d))
                  and os.path.exists(os.path.join(HERE, d, "meta.json")))


def load_program(name: str) -> Program:
    d = os.path.join(HERE, name)
    with open(os.path.join(d, "meta.json")) as fh:
        meta = json.load(fh)
    with open(os.path.join(d, "dense.ir")) as fh:
        dense = fh.read()
    local = sharding = None
    if os.path.exists(os.path.join(d, "local.ir")):
        with open(os.path.join(d, "local.ir")) as fh:
            local = fh.read()
        with open(os.path.join(d, "sharding.json")) as fh:
            sharding = json.load(fh)
    return Program(name, meta, dense, local, sharding)


def synthetic_inputs(module, seed: int = 0, scale: float = 0.02, func: str = "main") -> dict:
    """Deterministic N(0, scale^2) float32 inputs in signature order -- the
    same generator and draw order as the reference's `random_inputs`
    (interp.py:135-145), so a seed names the same arrays on every machine.
    scale 0.02 keeps deep transformer steps finite."""
    import numpy as np
    rng = np.random.default_rng(seed)
    f = module.func(func)
    return {n: (scale * rng.standard_normal(t.dims)).astype(np.float32) for n, t in f.args}


# benchmark workloads: BASELINE.json configs -> program per GPU count
WORKLOADS = {
    "c1": {"desc": "mlp_train(hidden_layers=1, batch=256, width=1024), BP",
           "scale": 0.25, "programs": {1: "c1_mlp_dense", 2: "c1_mlp_bp_B2"}},
    "c2": {"desc": "mini_transformer_train(blocks=8, batch=2048, d_model=1024, d_ff=4096), BP+MP",
           "scale": 0.02, "programs": {1: "c2_tf8_dense", 2: "c2_tf8_bp_B2", 4: "c2_tf8_bpmp_B2M2",
                                       8: "c2_tf8_bpmp_B2M4"}},
    "c3": {"desc": "mini_transformer_train(blocks=32, batch=8192, d_model=2048, d_ff=8192), BP+Z3",
           "scale": 0.02, "programs": {1: "c3_tf32_dense", 2: "c3_tf32_bpz3_B2", 4: "c3_tf32_bpz3_B4",
                                       8: "c3_tf32_bpz3_B8"},
           # the CPU evaluator cannot hold 32 blocks: its step time is
           # t(1 block) + 31 (t(2 blocks) - t(1 block)) at full width
           "cpu_extrap": {"blocks": 32, 1: ("c3_tf1_dense", "c3_tf2_dense"),
                          2: ("c3_tf1_bpz3_B2", "c3_tf2_bpz3_B2"), 4: ("c3_tf1_bpz3_B4", "c3_tf2_bpz3_B4"),
                          8: ("c3_tf1_bpz3_B8", "c3_tf2_bpz3_B8")}},
    "c4": {"desc": "unet_train(batch=128, 32x32, channels 64/256/512) U-Net analog (tools/unet_model.py), BP+Z2",
           "scale": 0.05, "programs": {1: "c4_unet_dense", 2: "c4_unet_bpz2_B2", 4: "c4_unet_bpz2_B4",
                                       8: "c4_unet_bpz2_B8"}},
    "c5": {"desc": "mini_transformer_train(blocks=8, batch=2048, d_model=1024, d_ff=4096), BP+MP+Z3+EMB",
           "scale": 0.02, "programs": {1: "c2_tf8_dense", 2: "c5_tf8_bpz3_B2", 4: "c5_tf8_bpmpz3_B2M2",
                                       8: "c5_tf8_bpmpz3emb_B2M2E2"}},
}
