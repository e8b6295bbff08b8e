"""One line per bench log: tag, n, config, samples/s, ms/step, e2e, per-class ms."""
import json
import sys

for path in sys.argv[1:]:
    line = None
    for l in open(path):
        l = l.strip()
        if l.startswith("{") and '"metric"' in l:
            line = json.loads(l)
    if line is None:
        print(path, "NO RESULT")
        continue
    r = line.get("roofline", {})
    sr = line.get("step_roofline", {})
    print(path.split("/")[-1], line["n_gpus"], line["config"].get("program"), round(line["value"]),
          round(line["ms_per_step"], 3), "e2e", round(line.get("e2e", {}).get("value", 0)),
          r.get("step_ms_by_class"), "gemm frac", round(r.get("frac", 0) or 0, 3),
          "step frac", round(sr.get("frac", 0) or 0, 3),
          "coll", (line.get("collectives_per_step") or {}).get("executed"),
          "clk", line.get("clocks", {}).get("sm_mhz"), line.get("clocks", {}).get("reasons"))
