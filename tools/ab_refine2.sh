#!/bin/bash
for lib in variants/libgpbo_prev.so paper_2403_08131_b200/libgpbo.so; do for r in 1 2; do
GPBO_LIB=$lib timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown_ms_per_step']; print('cfg3', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'refine', round(b['refine'],4))"
GPBO_LIB=$lib timeout 300 python bench.py --config 5 --steps 100 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown_ms_per_step']; print('cfg5', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'refine', round(b['refine'],4))"
done; done
