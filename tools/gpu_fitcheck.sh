#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fit" 2>&1 | tail -5
NOBENCH=1 bash tools/gpu_r2.sh
for c in 1 2 3 4; do for f in single cluster; do
GPBO_FIT=$f timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg${c}_$f.log 2>&1
grep "^{" gpurun_out/bench_cfg${c}_$f.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('cfg$c $f', '%.4g'%j['value'], round(j['ms_per_step'],4), 'refined', j['refined_per_step'], {k: round(v,4) for k,v in j['breakdown_ms_per_step'].items()})" || tail -3 gpurun_out/bench_cfg${c}_$f.log
done; done
