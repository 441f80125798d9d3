#!/bin/bash
# Profiling recipe for profiles/ (run on the GPU box from the repo root):
#   1. the bench command must exit 0 without ncu first;
#   2. launch list (gpu__time_duration per launch, clocks uncontrolled) of the same command;
#   3. one `--set full` capture of each hot kernel (a steady-state launch of the same command).
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu"
python bench.py $ARGS > "$OUT/pre_bench.log" 2>&1 || { echo "bench failed"; tail -20 "$OUT/pre_bench.log"; exit 1; }
tail -c 600 "$OUT/pre_bench.log"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py $ARGS --under-ncu > "$OUT/ncu_launches.log" 2>&1
echo "launch list rc=$?"
for k in k_fused_blocks k_zsweep_ring k_band_scan; do
    ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 2 -c 1 \
        -o "$OUT/full_$k" python bench.py $ARGS --under-ncu > "$OUT/ncu_full_$k.log" 2>&1
    echo "$k full capture rc=$?"
done
