#!/bin/bash
# A/B of the fit: variants/libgpbo_prev.so vs the tree's libgpbo.so (fit parity tests on the tree's)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ml2.py tests/test_gpu_append.py -m gpu -x -q -k "fit or ml2 or append" 2>&1 | tail -1
for c in ${CFGS:-2 3}; do for r in 1 2; do
for lib in variants/libgpbo_prev.so paper_2403_08131_b200/libgpbo.so; do
GPBO_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('cfg$c', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'fit', round(j['breakdown_ms_per_step']['fit'],4))"
done; done; done
