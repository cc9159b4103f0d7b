#!/bin/bash
# C1 (one 640x480 frame per batch) latency and stage times, plus C2 throughput, via bench.py's
# config measurements (no CPU baseline).
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/b.json 2>/tmp/b.err || { tail -5 /tmp/b.err; exit 1; }
python - <<'PY'
import json
d = json.load(open("/tmp/b.json")); c = d["configs"]
print("bench", d["value"], "gradhist", d["stages_ms"]["gradhist"]["ms"], "nms", d["stages_ms"]["nms"]["ms"], "ert", d["stages_ms"]["ert"]["ms"])
print("C1 latency", c["C1"]["latency_ms"], "e2e", c["C1"]["e2e"]["latency_ms"], "x4", c["C1"]["value_4_in_flight"])
print("   ", {k: v["ms"] for k, v in c["C1"]["stages_ms"].items()})
for k in ("C2", "C3", "C5"):
    print(k, c[k]["value"], "e2e", c[k]["e2e"]["value"], {s: v["ms"] for s, v in c[k]["stages_ms"].items()})
print("C4", c["C4"]["value"])
print("run", c["run"])
PY
