#!/bin/bash
# diagnostics: ncu full capture of the scoring kernel at cfg2/cfg3, then the clock64 trace (cfg2)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 3 -c 1 \
    -o gpurun_out/diag_score_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/diag_cfg2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 3 -c 1 \
    -o gpurun_out/diag_score_cfg3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/diag_cfg3.log 2>&1
GPBO_TC_TRACE=1 python -c "from paper_2403_08131_b200 import build as b; b.build()" > gpurun_out/trace_build.log 2>&1
timeout 120 python tools/trace_tc.py 100000 > gpurun_out/trace.txt 2>&1
tail -2 gpurun_out/trace.txt
