#!/bin/bash
# usage (under gpurun): tools/ab.sh "<cfgs>" <variant letters...>  (variants/lib<V>.so; "0" = package lib)
cfgs=$1; shift
for v in "$@"; do
  for c in $cfgs; do
    if [ "$v" = "0" ]; then lib=""; else lib=variants/lib$v.so; fi
    GPBO_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${v}_$c.log 2>&1
    echo "$v cfg$c" $(grep -o '"fast": [0-9.]*' gpurun_out/ab_${v}_$c.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${v}_$c.log) $(grep -o '"idx": [0-9]*' gpurun_out/ab_${v}_$c.log)
  done
done
