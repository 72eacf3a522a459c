#!/bin/bash
# A/B of the scoring kernel: variants/libgpbo_prev.so vs the tree's libgpbo.so (same box)
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_soundness.py -q -x 2>&1 | tail -2
for c in ${CFGS:-2 3}; do for r in 1 2; do
for lib in variants/libgpbo_prev.so paper_2403_08131_b200/libgpbo.so; do
GPBO_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('cfg$c', '$lib'.split('/')[-1], round(j['ms_per_step'],4), 'fast', round(j['breakdown_ms_per_step']['fast'],4), 'frac', round(j['roofline']['frac'],4))"
done; done; done
