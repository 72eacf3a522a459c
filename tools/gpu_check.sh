#!/bin/bash
# usage (under gpurun): tools/gpu_check.sh [configs...]  -> gpu tests + smoke + bench sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in ${@:-1 2 3}; do
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
