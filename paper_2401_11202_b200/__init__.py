"""paper_2401_11202_b200: B200-native evaluator for PartIR-partitioned programs.

Drop-in replacement for the reference's partitioned-program evaluator
(`spindle.spmd_interp.spmd_interpret`, /root/reference/pkg/src/spindle/
spmd_interp.py:157-197).  Localized SPMD modules (from the reference's
unchanged tactic API: Partitioner / lower_to_spmd / localize) run on B200s:
hand-written sm_100a kernels behind a C-ABI (include/spindle_b200.h), in-GPU
group collectives for co-located mesh devices, NCCL across GPUs.
"""
from .evaluator import DivergenceError, EvalError, interpret, relative_error, spmd_interpret
from .ir import Mesh, Module, ShardingSpec, collective_counts, compute_flops, parse_module
from .programs import Program, list_programs, load_program

__all__ = [
    "spmd_interpret", "interpret", "DivergenceError", "EvalError", "relative_error",
    "parse_module", "ShardingSpec", "Mesh", "Module", "collective_counts", "compute_flops",
    "Program", "load_program", "list_programs",
]
