"""The drop-in calls' compiled-plan cache, host logic only:
fingerprints identify programs structurally (our IR objects and the
reference's give the same key; any change to an op, type, attribute or the
mesh changes it), and the LRU honours its entry and byte bounds."""
import pytest

from conftest import golden_cases
from paper_2401_11202_b200 import evaluator as E
from paper_2401_11202_b200.ir import parse_module


def test_fingerprint_structural():
    case = next(c for c in golden_cases() if c["key"] == "rule_rs_raw")
    a = parse_module(case["local_ir"])
    b = parse_module(case["local_ir"])
    assert E.fingerprint(a) == E.fingerprint(b)
    text = case["local_ir"]
    c = parse_module(text.replace("4x4", "4x4", 1))
    assert E.fingerprint(c) == E.fingerprint(a)
    d = parse_module(text.replace("mesh {K:4}", "mesh {K:2}")) if "mesh {K:4}" in text else None
    if d is not None:
        assert E.fingerprint(d) != E.fingerprint(a)


def test_fingerprint_matches_reference_objects():
    spindle = pytest.importorskip("spindle")
    from spindle.parser import parse_module as ref_parse
    n = 0
    for case in golden_cases()[:30]:
        text = case.get("local_ir") or case.get("dense_ir")
        try:
            ref = ref_parse(text)
        except Exception:          # hand-built layouts the reference's parser rejects (repeated axes)
            continue
        assert E.fingerprint(parse_module(text)) == E.fingerprint(ref), case["key"]
        n += 1
    assert n >= 10


def test_fingerprint_sensitive_to_attrs_and_types():
    t1 = ("func @main(%x: tensor<8x4xf32>) -> tensor<4x8xf32> {\n"
          "  %t = transpose %x {perm = [1, 0]} : tensor<4x8xf32>\n  return %t\n}\n")
    t2 = t1.replace("xf32", "xi32")
    t3 = t1.replace("8x4xf32", "16x4xf32").replace("4x8xf32", "4x16xf32")
    fps = {E.fingerprint(parse_module(t)) for t in (t1, t2, t3)}
    assert len(fps) == 3


class _FakeEx:
    def __init__(self, nbytes):
        self.dev_stride, self.ndev = nbytes, 1
        self.closed = False

    def close(self):
        self.closed = True


def test_plan_cache_lru_bounds(monkeypatch):
    monkeypatch.setenv("SPX_PLAN_CACHE", "2")
    monkeypatch.setenv("SPX_PLAN_CACHE_BYTES", str(100))
    c = E.PlanCache()
    a, b, d = _FakeEx(40), _FakeEx(40), _FakeEx(40)
    assert c.put("a", a) and c.put("b", b)
    assert c.get("a") is a                 # a is now most recent
    assert c.put("d", d)                   # evicts b (LRU), entry bound 2
    assert b.closed and not a.closed and c.get("b") is None
    big = _FakeEx(1000)
    assert not c.put("big", big)           # larger than the byte bound: not cached
    assert c.get("big") is None
    monkeypatch.setenv("SPX_PLAN_CACHE", "0")
    e = _FakeEx(1)
    assert not c.put("e", e)               # caching disabled
    c.clear()
    assert a.closed and d.closed
