# A/B of the band scan's staging (HSZG_BS_NBUF: 2 = double-buffered, unset = one buffer where it adds a CTA per SM)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_api.py tests/test_gpu_configs.py tests/test_gpu_pipeline.py tests/test_gpu_golden.py tests/test_gpu_streaming.py -x -q -m gpu > gpurun_out/nbuf_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/nbuf_tests.log
for nb in 2 0; do
HSZG_BS_NBUF=$nb python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact > gpurun_out/nbuf_$nb.log 2>&1
python - <<P
import json
l=[x for x in open('gpurun_out/nbuf_$nb.log') if x.startswith('{')]
d=json.loads(l[-1]); print('NBUF=$nb step', d['ms_per_step'], d['roofline']['frac'])
for x in d.get('rows',{}).get('rows',[]):
    if x['kind']=='HSZP_ND' and any(s in x['row'] for s in ('A3','N1 variance at stage 3','A13 gradient at stage 3','A7')): print('NBUF=$nb', x['row'], x['api_ms'], x['kernel_ms'], x['kernels_us'])
P
done
