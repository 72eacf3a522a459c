#!/bin/bash
# A/B of two library builds on one box: ab2.sh LIB_A LIB_B [configs] (bench fast-phase + step)
A=${1:-variants/libgpbo_base.so}; B=${2:-paper_2403_08131_b200/libgpbo.so}; CF=${3:-"2 3"}
for c in $CF; do for r in 1 2; do for lib in $A $B; do
GPBO_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline $EXTRA 2>&1 | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); b=j['breakdown_ms_per_step']; print('cfg$c', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'fast', round(b['fast'],4), 'refine', round(b.get('refine',0),4), 'frac', round(j['roofline']['frac'],4), 'refined', j.get('refined_per_step'), 'idx_ok', j.get('oracle_idx_match'))"
done; done; done
