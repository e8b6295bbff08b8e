"""tools/timeline.py's analysis of a traced multi-stream run (CPU): stall
attribution on a synthetic trace, and the committed N=4 C2 trace before the
scheduling fix reproduces the stall DESIGN.md §5 reports."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from timeline import analyse  # noqa: E402


def test_stall_attributed_to_the_last_finishing_wait():
    # main: gemm [0,1], then ew waits for a peer collective on stream 2 that ends at 3
    cls = ["gemm", "peer", "copy", "ew"]
    stream = [0, 2, 2, 0]
    ready = [0.0, 1.0, 0.0, 3.0]
    end = [1.0, 3.0, 0.5, 3.5]
    waits = [[], [0], [], [1, 2]]
    out = analyse(cls, stream, ready, end, waits)
    assert out["span_ms"] == 3.5
    assert out["main_stall_ms"] == 2.0
    assert out["main_stall_by_cause"] == {"peer@s2": [2.0, 1]}
    assert out["busy_ms_by_stream"] == {0: 1.5, 2: 2.5}


def test_committed_c2_trace_shows_the_critical_allreduce_stall():
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_timeline_c2_n4_before.json")))
    out = analyse(d["cls"], d["stream"], d["ready"], d["end"], d["waits"])
    causes = out["main_stall_by_cause"]
    assert "peer@s2" in causes and causes["peer@s2"][0] > 2.0      # ms of a ~5.3 ms step
    after = json.load(open(os.path.join(ROOT, "profiles", "r02_timeline_c2_n4_after.json")))
    out2 = analyse(after["cls"], after["stream"], after["ready"], after["end"], after["waits"])
    assert out2["span_ms"] < out["span_ms"]
