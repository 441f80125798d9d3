#!/bin/bash
# A/B timing of two source trees on one box (a Python + library change): ab/head (git archive of HEAD with
# its own libhszg.so) vs the working tree, alternating, 2 rounds each.
ARGS=${ARGS:-"--steps 5 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact --rows"}
mkdir -p gpurun_out
for round in 1 2; do
  for tree in ab/head .; do
    tag=$( [ "$tree" = "." ] && echo work || echo head )
    (cd $tree && timeout 300 python bench.py $ARGS --detail $OLDPWD/gpurun_out/abt_${tag}_$round.json) > gpurun_out/abt_${tag}_$round.log 2>&1
    python -c "
import json
d=json.load(open('gpurun_out/abt_${tag}_$round.json'))
print('$tag', $round, {k:round(v['ms'],2) for k,v in d['kernels'].items()})"
    grep -h ms_per_step gpurun_out/abt_${tag}_$round.log | python -c "
import sys,json
for l in sys.stdin:
    l=l[l.index('{'):]; d=json.loads(l); print('   step', d['ms_per_step'], 'hszp-nd frac', d['roofline']['frac'], 'hszx-nd', d['roofline']['other_ops']['hszx-nd']['frac'])"
  done
done
