#!/bin/bash
# round-end measurements (under gpurun): profiles + per-config bench lines + config-5 replay
tag=${1:-r01f}
bash tools/profile_round.sh $tag > /dev/null 2>&1
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 $( [ $c != 2 ] && echo --no-cpu-baseline ) > gpurun_out/${tag}_bench_cfg$c.log 2>&1
  grep '^{' gpurun_out/${tag}_bench_cfg$c.log > gpurun_out/${tag}_bench_cfg$c.json
  python -c "import json; j=json.load(open('gpurun_out/${tag}_bench_cfg$c.json')); print($c, '%.4g'%j['value'], '%.3f'%j['ms_per_step'], '%.4g'%j['e2e']['value'], round(j['roofline']['frac'],4), j['config']['scoring'], {k: round(v,4) for k,v in j['breakdown_ms_per_step'].items()})"
done
timeout 300 python tools/replay_bench.py > gpurun_out/${tag}_replay_cfg5.json 2>&1; tail -1 gpurun_out/${tag}_replay_cfg5.json
ls gpurun_out/${tag}_* | head -30
