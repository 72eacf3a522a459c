#!/bin/bash
# Round-2 profiles for profiles/ (under gpurun): the ncu launch list of the default bench step,
# full ncu captures of every kernel that matters, per-config bench lines, the reference arm, the
# config-5 replay and the Table III replay.  usage: tools/profile_r02.sh <tag>
tag=${1:-r02}
o=gpurun_out
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader > $o/${tag}_gpu.txt
# bench lines first (clean clocks, no profiler)
timeout 600 python bench.py --no-other-configs > $o/${tag}_bench_cfg2.json 2> $o/${tag}_bench_cfg2.err
timeout 900 python bench.py --impl reference > $o/${tag}_reference_cfg2.json 2>&1
for c in 1 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $o/${tag}_bench_cfg$c.json 2> $o/${tag}_bench_cfg$c.err
done
timeout 600 python bench.py --config 4 --scaling strong --steps 20 --warmup 5 --no-cpu-baseline > $o/${tag}_bench_cfg4_strong.json 2>&1
for c in 2 4; do
  timeout 600 python bench.py --config $c --layout bo --steps 10 --warmup 3 --no-cpu-baseline > $o/${tag}_bench_cfg${c}_bo.json 2>&1
done
timeout 900 python bench.py --config 5 --steps 200 --warmup 3 > $o/${tag}_bench_cfg5.json 2> $o/${tag}_bench_cfg5.err
timeout 600 python tools/replay_bench.py > $o/${tag}_replay_cfg5.json 2>&1
rm -f $o/${tag}_posterior_bench.jsonl
for c in 2 3 4; do timeout 300 python tools/posterior_bench.py $c >> $o/${tag}_posterior_bench.jsonl 2>&1; done
# launch list of the default step (cold-cache, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $o/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs \
    > $o/${tag}_launches_bench.log 2>&1
cap() {  # name regex args...
  local name=$1 re=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s 3 -c 1 \
      -o $o/${tag}_$name python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs "$@" \
      > $o/${tag}_$name.log 2>&1
}
cap score_tc 'score_tc_kernel'
cap score_tc_cfg3 'score_tc_kernel' --config 3
cap score_tcs 'score_tcs_kernel' --config 4
cap fit 'fit_kernel' 
cap fit_cluster 'fit_cluster_kernel' --config 4
cap refine 'refine' 
cap gram 'gram_kernel'
cap pack 'pack_tc'
cap mean64 'mean64' --layout bo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:posterior64 -s 2 -c 1 \
    -o $o/${tag}_posterior64 python tools/posterior_bench.py 2 65536 > $o/${tag}_posterior64.log 2>&1
ls -la $o/${tag}_*
