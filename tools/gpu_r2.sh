#!/bin/bash
# round-2 check (under gpurun): all gpu tests, smoke, default bench line (+ cpu baseline)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
if [ -z "$NOBENCH" ]; then
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
grep '^{' gpurun_out/bench_default.log > gpurun_out/bench_default.json; tail -c 3000 gpurun_out/bench_default.log
fi
