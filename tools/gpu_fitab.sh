#!/bin/bash
# fit change check: fit parity tests, then the config 2 / 3 step breakdown
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fit" 2>&1 | tail -1
for c in 2 3; do for r in 1 2; do
timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('cfg$c', round(j['ms_per_step'],4), {k: round(v,4) for k,v in j['breakdown_ms_per_step'].items()})"
done; done
