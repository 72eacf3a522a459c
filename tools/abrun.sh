for v in A B C; do
  GPBO_LIB=variants/lib$v.so timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
  echo $v $(grep -o '"fast": [0-9.]*' gpurun_out/bench_$v.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_$v.log)
done
