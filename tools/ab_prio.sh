# A/B: persistent band-scan grid (HSZG_BAND_CTAS) x side-stream priority (HSZP_ND overlap experiments)
mkdir -p gpurun_out
for round in 1; do
 for cfg in "P 1 -1 64" "P 1 -1 128" "P 1 -1 32"; do
  set -- $cfg
  tag=$1_c$2_p$3_w$4
  HSZG_BAND_CTAS=$2 HSZG_SIDE_PRIORITY=$3 HSZG_LIB=ab/lib_$1.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --window $4 --detail gpurun_out/abp_${tag}.json ${EXTRA} > gpurun_out/abp_${tag}_$round.log 2>&1
  echo "$tag $round $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/abp_${tag}_$round.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/abp_${tag}_$round.log | head -2 | tr '\n' ' ')"
 done
done
