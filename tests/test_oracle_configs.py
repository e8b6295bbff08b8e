"""Pin the oracle at the BASELINE configurations' sizes: the oracle
restatement and the reference's own evaluator (imported from
/root/reference, so this runs in the build container and skips elsewhere)
produce bit-identical outputs on the config programs the GPU parity tests
(tests/test_config_parity.py) compare against -- full width, the configs'
own meshes and tactics, reduced depth where the reference cannot hold the
full model."""
import numpy as np
import pytest

spindle = pytest.importorskip("spindle")

from oracle import spmd_oracle as O  # noqa: E402
from paper_2401_11202_b200.programs import load_program, synthetic_inputs  # noqa: E402


@pytest.mark.parametrize("name,mode,scale", [
    ("c1_mlp_bp_B2", "spmd", 0.25),
    ("c1_mlp_dense", "dense", 0.25),
    ("c2_tf1_bpmp_B2M4", "spmd", 0.02),
    ("c5_tf1_bpmpz3emb_B2M2E2", "spmd", 0.02),
    ("c3_tf1_dense", "dense", 0.02),
    ("c4_unet_bpz2_B8", "spmd", 0.05),
])
def test_oracle_matches_reference_at_config_size(name, mode, scale):
    from spindle.interp import interpret as ref_interpret
    from spindle.interp import random_inputs as ref_random_inputs
    from spindle.parser import parse_module as ref_parse
    from spindle.spmd import ShardingSpec as RefSpec
    from spindle.spmd_interp import spmd_interpret as ref_spmd
    prog = load_program(name)
    ins = synthetic_inputs(prog.dense, seed=0, scale=scale)
    ref_ins = ref_random_inputs(ref_parse(prog.dense_text), seed=0, scale=scale)
    for n in ins:                                  # same generator, same draws
        np.testing.assert_array_equal(ins[n], ref_ins[n])
    if mode == "spmd":
        got = O.spmd_interpret(prog.local, prog.sharding, ins)
        want = ref_spmd(ref_parse(prog.local_text), RefSpec.from_json(prog.sharding_json), ref_ins)
    else:
        got = O.interpret(prog.dense, ins)
        want = ref_interpret(ref_parse(prog.dense_text), ref_ins)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g.dtype == w.dtype and g.shape == w.shape
        np.testing.assert_array_equal(g, w)
