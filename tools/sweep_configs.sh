#!/bin/bash
# usage: tools/sweep_configs.sh  (under gpurun) -> one bench line per config in gpurun_out/sweep_*.json
mkdir -p gpurun_out
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_cfg$c.log 2>&1
  grep '^{' gpurun_out/sweep_cfg$c.log > gpurun_out/sweep_cfg$c.json
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    j = json.loads(open(f"gpurun_out/sweep_cfg{c}.json").read())
    print("cfg", c, "value %.4g ms/step %.3f e2e %.4g frac %.4f %s" % (j["value"], j["ms_per_step"], j["e2e"]["value"], j["roofline"]["frac"], j["config"]["scoring"]),
          {k: round(v, 4) for k, v in j["breakdown_ms_per_step"].items()})
except Exception as e:
    print("cfg", c, "FAILED", e, open(f"gpurun_out/sweep_cfg{c}.log").read()[-1500:])
PY
done
