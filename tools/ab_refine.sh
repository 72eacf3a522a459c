#!/bin/bash
# A/B of the refine: step and refine time per config (tree vs variants/libgpbo_prev.so)
for c in ${CFGS:-2 4}; do for r in 1 2; do for lib in variants/libgpbo_prev.so paper_2403_08131_b200/libgpbo.so; do
GPBO_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown_ms_per_step']; print('cfg$c', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'refine', round(b['refine'],4), j['refined_per_step'])"
done; done; done
