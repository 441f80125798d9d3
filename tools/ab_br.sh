# A/B: HSZP_ND band height of the band scan (config 5)
for round in 1 2; do
 for br in ${BRS:-64 128 256}; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --band-rows $br > gpurun_out/abbr_${br}_$round.log 2>&1
  echo "br $br $round $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/abbr_${br}_$round.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/abbr_${br}_$round.log | head -1)"
 done
done
