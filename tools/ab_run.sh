#!/bin/bash
# A/B timing on one box: alternate the libraries given as arguments (paths), 2 rounds each.
ARGS=${ARGS:-"--steps 5 --warmup 3 --no-e2e --no-cpu"}
mkdir -p gpurun_out
for round in 1 2; do
  for lib in "$@"; do
    tag=$(basename $lib .so)
    HSZG_LIB=$lib timeout 300 python bench.py $ARGS --detail gpurun_out/ab_${tag}_$round.json > gpurun_out/ab_${tag}_$round.log 2>&1
    python -c "
import json
d=json.load(open('gpurun_out/ab_${tag}_$round.json'))
print('$tag', $round, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
  done
done
