#!/bin/bash
# usage: tools/bench_brief.sh [bench args...]  -> prints value and per-kernel breakdown
timeout 300 python bench.py "$@" > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
for line in open("gpurun_out/bench.log"):
    line = line.strip()
    if line.startswith("{"):
        j = json.loads(line)
        print("value %.4g  ms/step %.3f  e2e %.4g  frac %.4f  refined %s" % (j["value"], j["ms_per_step"], j["e2e"]["value"], j["roofline"]["frac"], j.get("refined_per_step")))
        print("breakdown", {k: round(v, 4) for k, v in j["breakdown_ms_per_step"].items()})
        break
else:
    print(open("gpurun_out/bench.log").read()[-3000:])
PY
