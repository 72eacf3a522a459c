#!/bin/bash
# Profiles for profiles/ (run under gpurun): the launch list of a short config-2 bench run, and
# full ncu captures of the scoring kernels (config 2: score_tc, config 4: score_tcs), the fit
# and the refine kernel.  usage: tools/profile_round.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 3 -c 1 \
    -o gpurun_out/${tag}_score_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_score_tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_tcs_kernel -s 3 -c 1 \
    -o gpurun_out/${tag}_score_tcs python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_score_tcs.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fit_kernel -s 3 -c 1 \
    -o gpurun_out/${tag}_fit python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_fit.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:refine -s 3 -c 1 \
    -o gpurun_out/${tag}_refine python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_refine.log 2>&1
ls -la gpurun_out/${tag}_*
