set -x
for v in A B C; do
  GPBO_LIB=variants/lib$v.so timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
  grep -o '"breakdown_ms_per_step": {[^}]*}' gpurun_out/bench_$v.log; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_$v.log
done
GPBO_LIB=variants/libA.so timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
