#!/bin/bash
# A/B of posterior64 variants: tools/posterior_bench.py per library, configs 2 3 4
for lib in paper_2403_08131_b200/libgpbo.so variants/libgpbo_*.so; do for c in ${CFGS:-2 3 4}; do
GPBO_LIB=$lib timeout 120 python tools/posterior_bench.py $c 2>&1 | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib'.split('/')[-1], 'cfg$c', round(j['posterior']['ms'],4), 'x%.2f' % j['posterior_over_argmax'])"
done; done
