#!/bin/bash
# Round-2 evidence run (one box): GPU tests, the driver's bench command, the reference arm, ncu captures
# of the API kernels changed this round (tools/profile_rows.py, config 4) and of the exact-fp32 (table)
# emitter kernels in the config-5 step.  Outputs in gpurun_out/ (copy the summaries to profiles/).
set -u
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/t_gpu_final.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/t_gpu_final.log
python bench.py --steps 20 --warmup 5 > $O/bench_final.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_final.log 2>&1; echo "ref rc=$?"
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include 'rows/' \
    -k regex:'k_(reduce|fused|hszp_tile|wt_)' -o $O/api_final \
    python tools/profile_rows.py --only mean2 var3 grad3 lap3 stage3 > $O/ncu_api_final.log 2>&1
echo "ncu api rc=$?"
ncu --csv --page raw -i $O/api_final.ncu-rep > $O/api_final_raw.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:'k_zsweep_ring|k_fused_blocks' --launch-skip 40 -c 2 \
    -o $O/exact_final python bench.py --steps 1 --warmup 3 --exact-fp32 --no-e2e --no-cpu --no-parity --no-exact \
    --rows --under-ncu > $O/ncu_exact_final.log 2>&1
echo "ncu exact rc=$?"
ncu --csv --page raw -i $O/exact_final.ncu-rep > $O/exact_final_raw.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact --rows --under-ncu > $O/ncu_launches_final.log 2>&1
echo "launch list rc=$?"
