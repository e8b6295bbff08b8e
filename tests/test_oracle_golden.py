"""Pin the oracle restatement to the reference's own outputs (golden vectors
produced by tests/golden/make_golden.py running /root/reference)."""
import numpy as np
import pytest

from conftest import case_expected, case_inputs, golden_cases, golden_outputs
from oracle import spmd_oracle as O
from paper_2401_11202_b200.ir import ShardingSpec, collective_counts, compute_flops, parse_module

CASES = golden_cases()


def test_random_inputs_fingerprint():
    """random_inputs (interp.py:135-145) draws identically to the reference."""
    m = parse_module(next(c for c in CASES if c["key"] == "acc_mlp_bp")["dense_ir"])
    want = golden_outputs()["fingerprint/random_inputs_mlp_s3/x"]
    np.testing.assert_array_equal(O.random_inputs(m, seed=3)["x"], want)


@pytest.mark.parametrize("case", [c for c in CASES if "local_ir" in c], ids=lambda c: c["key"])
def test_oracle_spmd_matches_reference(case):
    m = parse_module(case["local_ir"])
    spec = ShardingSpec.from_json(case["sharding"])
    if "counts" in case:
        assert collective_counts(m) == case["counts"]
    if "compute_flops" in case:
        assert compute_flops(m) == case["compute_flops"]
    base = parse_module(case["dense_ir"]) if "dense_ir" in case else m
    for s in case["seeds"]:
        ins = case_inputs(case, base, s)
        if case.get("error") == "DivergenceError":
            with pytest.raises(O.DivergenceError):
                O.spmd_interpret(m, spec, ins)
            continue
        got = O.spmd_interpret(m, spec, ins)
        for g, w in zip(got, case_expected(case, s, "spmd")):
            np.testing.assert_array_equal(g, w)      # bit-exact: same numpy ops


@pytest.mark.parametrize("case", [c for c in CASES if "dense_ir" in c], ids=lambda c: c["key"])
def test_oracle_dense_matches_reference(case):
    m = parse_module(case["dense_ir"])
    for s in case["seeds"]:
        ins = case_inputs(case, m, s)
        got = O.interpret(m, ins)
        for g, w in zip(got, case_expected(case, s, "dense")):
            np.testing.assert_array_equal(g, w)
