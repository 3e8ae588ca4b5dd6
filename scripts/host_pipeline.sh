#!/bin/bash
# bench value + host pool occupancy per step (fill / gaps / drain), optional env prefix
python bench.py --no-cpu-baseline "$@" > gpurun_out/hp.log 2>&1
python - <<'PY'
import json
l = [x for x in open("gpurun_out/hp.log") if x.startswith("{")][-1]
d = json.loads(l)
h = d["host_pipeline_ms_per_step"]
print(round(d["value"], 1), round(d["e2e"]["value"], 1), round(d["ms_per_step"], 2),
      {k: round(v, 2) for k, v in h.items()}, round(d["roofline"]["frac"], 3))
PY
