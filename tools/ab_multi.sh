#!/bin/bash
# A/B over every variants/libgpbo_*.so plus the tree's library: step and fast phase per config
for c in ${CFGS:-2 3}; do for r in 1 2; do
for lib in paper_2403_08131_b200/libgpbo.so variants/libgpbo_*.so; do
GPBO_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown_ms_per_step']; print('cfg$c', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'fast', round(b['fast'],4), 'fit', round(b['fit'],4))"
done; done; done
