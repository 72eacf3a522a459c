#!/bin/bash
for c in 2 4; do for lib in paper_2403_08131_b200/libgpbo.so variants/libgpbo_*.so; do for r in 1 2; do
GPBO_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown_ms_per_step']; print('cfg$c', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'pack', round(b['pack'],4), 'fast', round(b['fast'],4))"
done; done; done
