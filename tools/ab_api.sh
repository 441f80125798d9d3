# A/B of API-level stage / stats calls (config 4) and of the bench step, for the libraries given (paths)
for lib in "$@"; do
  echo "== $(basename $lib .so)"
  HSZG_LIB=$lib timeout 400 python tools/ab_stage3.py --stats --reps 10 2>&1 | grep kind | sed "s/BR=- //" | cut -c1-150
  HSZG_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact --rows \
      --detail gpurun_out/abapi_$(basename $lib .so).json > gpurun_out/abapi_$(basename $lib .so).log 2>&1
  echo "step $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/abapi_$(basename $lib .so).log | head -1)"
done
