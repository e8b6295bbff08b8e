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
