#!/bin/bash
# compute-sanitizer passes over a selection of the GPU tests (small shapes: the tools replay every
# access).  usage (under gpurun): tools/sanitize.sh
mkdir -p gpurun_out
sel='test_fit_matches_oracle and (1-1 or 9-3 or 33-8 or 224-12) or test_posterior_matches_oracle and (n17 or cfg1) or test_empty_and_single or test_exact_tie or test_nan_candidate'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$sel" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
  python -m pytest tests/test_gpu_append.py tests/test_gpu_ml2.py tests/test_gpu_edge.py -q -p no:cacheprovider -k "not cfg2 and not config3" > gpurun_out/sanitize_memcheck2.log 2>&1
echo "memcheck2 rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_memcheck2.log | tr '\n' ' ')"
