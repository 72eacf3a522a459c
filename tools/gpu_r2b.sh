#!/bin/bash
mkdir -p gpurun_out
NOBENCH=1 bash tools/gpu_r2.sh
for c in 2 4; do for l in uniform bo; do
timeout 600 python bench.py --config $c --layout $l --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg${c}_$l.log 2>&1
grep "^{" gpurun_out/bench_cfg${c}_$l.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['config']['workload'][:5], j['config']['layout'], '%.4g'%j['value'], round(j['ms_per_step'],4), 'refined', j['refined_per_step'], {k: round(v,4) for k,v in j['breakdown_ms_per_step'].items()})" || tail -5 gpurun_out/bench_cfg${c}_$l.log
done; done
bash tools/t3_sweep.sh
