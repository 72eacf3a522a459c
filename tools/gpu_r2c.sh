#!/bin/bash
# re-entry check: full GPU suite + bench lines of configs 2/3/4 at HEAD
o=gpurun_out; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/r2c_gputests.log 2>&1; echo "pytest rc $?" >> $o/r2c_gputests.log
timeout 300 python bench.py --no-cpu-baseline > $o/r2c_cfg2.json 2> $o/r2c_cfg2.err
for c in 3 4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $o/r2c_cfg$c.json 2> $o/r2c_cfg$c.err; done
tail -3 $o/r2c_gputests.log
