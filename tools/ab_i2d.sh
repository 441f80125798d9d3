for lib in ab/lib_HEAD.so ab/lib_i2d.so; do
  HSZG_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity --rows > gpurun_out/abx_$(basename $lib .so).log 2>&1
  echo "$lib $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/abx_$(basename $lib .so).log | head -1) exact: $(grep -o '"exact_fp32": {[^}]*}' gpurun_out/abx_$(basename $lib .so).log | head -1)"
  HSZG_LIB=$lib timeout 300 python tools/ab_stage3.py --reps 20 2>&1 | grep kind
done
