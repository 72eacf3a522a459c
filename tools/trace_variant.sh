#!/bin/bash
# usage (under gpurun): tools/trace_variant.sh <cfg> <DEFINE...> -> gpurun_out/trace_v_cfg<cfg>.txt
cfg=$1; shift
defs=""
for d in "$@"; do defs="$defs'$d',"; done
python -c "
import sys; sys.path.insert(0,'.')
from paper_2403_08131_b200 import build as b
print(b.build(defines=('GPBO_TC_TRACE',$defs), out='variants/libTR.so'))" > gpurun_out/trace_vbuild.log 2>&1
GPBO_LIB=variants/libTR.so timeout 120 python tools/trace_tc.py 1000000 $cfg > gpurun_out/trace_v_cfg$cfg.txt 2>&1
tail -1 gpurun_out/trace_v_cfg$cfg.txt
