#!/bin/bash
# posterior kernel check: the posterior-touching GPU tests, then its throughput per config
o=gpurun_out; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_suggest.py -m gpu -x -q -k "posterior or T1 or t1 or nan or Posterior" > $o/post_tests.log 2>&1; echo "rc $?" >> $o/post_tests.log
for c in 2 3 4; do timeout 300 python tools/posterior_bench.py $c >> $o/post_bench.jsonl 2>&1; done
tail -3 $o/post_tests.log; cat $o/post_bench.jsonl
