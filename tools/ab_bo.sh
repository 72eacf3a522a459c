#!/bin/bash
# A/B of the precise-mean tier: config 2 / 4 BO layouts per library (tree + variants)
for c in 2 4; do for lib in paper_2403_08131_b200/libgpbo.so variants/libgpbo_*.so; do
GPBO_LIB=$lib timeout 300 python bench.py --config $c --layout bo --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown_ms_per_step']; print('cfg$c bo', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'mean', round(b['mean'],4), 'refined', j['refined_per_step'])"
done; done
