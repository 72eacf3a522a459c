#!/bin/bash
# ncu --set full of the scoring kernel for two builds: ncu_ab.sh LIB_A LIB_B [bench args]
A=$1; B=$2; shift 2
mkdir -p gpurun_out
for lib in $A $B; do
  n=$(basename $lib .so)
  GPBO_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 3 -c 1 \
    -o gpurun_out/ab_$n -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ab_$n.log 2>&1
  echo "== $n"; python tools/ncu_summary.py gpurun_out/ab_$n.ncu-rep 12 2>&1 | head -40
  ncu -i gpurun_out/ab_$n.ncu-rep --page source --csv --print-source=sass 2>/dev/null | python tools/ncu_stalls.py 12
done
