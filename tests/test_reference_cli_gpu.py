"""The reference's own parity harness (`spindle verify`, cli.py:139-178) with
the B200 evaluator bound in through the plugin rebinding of INTEGRATION.md:
clean schedules verify (exit 0) and the harness self-test -- an all_reduce
emptied of its axes -- is caught with exit 3 (test_cli.py:155-160), on the
GPU.  Needs the reference package (skipped where it is absent)."""
import pytest

spindle = pytest.importorskip("spindle")


@pytest.fixture
def b200_plugin(monkeypatch):
    import spindle.cli
    import spindle.spmd_interp
    import paper_2401_11202_b200 as b200
    calls = []

    def spmd_interpret(*a, **k):
        calls.append(1)
        return b200.spmd_interpret(*a, **k)
    monkeypatch.setattr(spindle.spmd_interp, "spmd_interpret", spmd_interpret)
    monkeypatch.setattr(spindle.cli, "spmd_interpret", spmd_interpret)
    return calls


@pytest.mark.gpu
@pytest.mark.parametrize("argv", [
    ["--module", "chain", "--mesh", "B:4,M:2", "--schedule", "bp,mp"],
    ["--module", "mlp", "--mesh", "B:2", "--schedule", "bp", "--layers", "2"],
    ["--module", "transformer", "--mesh", "B:2,M:2", "--schedule", "bp,mp,z3"],
])
def test_reference_verify_on_b200(b200_plugin, argv, capsys):
    from spindle.cli import main
    code = main(["verify", *argv, "--trials", "2"])
    out = capsys.readouterr()
    assert code == 0, out.err
    assert out.out.startswith("ok: 2 trials")
    assert len(b200_plugin) == 2


@pytest.mark.gpu
def test_reference_self_test_corrupt_caught_on_b200(b200_plugin, capsys):
    from spindle.cli import main
    code = main(["verify", "--module", "chain", "--mesh", "B:4,M:2", "--schedule", "bp,mp",
                 "--trials", "2", "--self-test-corrupt"])
    assert code == 3
    assert "FAIL" in capsys.readouterr().err
    assert b200_plugin
