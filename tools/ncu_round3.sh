#!/bin/bash
# Round-2 final evidence run (one box, fourth session): GPU tests, the driver's bench command, the reference arm,
# the configs 1-4 row table, and the launch list of the config-5 step.  Outputs in gpurun_out/.
set -u
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/t_gpu_final.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/t_gpu_final.log
python bench.py --steps 20 --warmup 5 > $O/bench_final.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_final.log 2>&1; echo "ref rc=$?"
timeout 1200 python bench_rows.py --configs 1 2 3 4 --out $O/rows_final.json > $O/rows_final.log 2>&1; echo "rows rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact --rows --under-ncu > $O/ncu_launches_final.log 2>&1
echo "launch list rc=$?"
