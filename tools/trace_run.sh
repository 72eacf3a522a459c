#!/bin/bash
# usage (under gpurun): tools/trace_run.sh <cfg...> -> gpurun_out/trace_cfg<c>.txt (clock64 trace build)
mkdir -p gpurun_out
GPBO_TC_TRACE=1 python -c "from paper_2403_08131_b200 import build as b; b.build()" > gpurun_out/trace_build.log 2>&1
for c in "$@"; do
  timeout 120 python tools/trace_tc.py 1000000 $c > gpurun_out/trace_cfg$c.txt 2>&1
  tail -1 gpurun_out/trace_cfg$c.txt
done
