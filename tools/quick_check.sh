# quick A/B loop: pipeline / headline / API tests, then the config-5 step and the config-4 rows
mkdir -p gpurun_out
python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_headline.py tests/test_gpu_api.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/qc_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/qc_tests.log
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact > gpurun_out/qc_bench.log 2>&1; echo "bench rc=$?"
python - <<P
import json
l=[x for x in open('gpurun_out/qc_bench.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('step', d['ms_per_step'], 'frac', r['frac'], {k:v.get('ms_per_step') for k,v in r.get('kernels',{}).items()}, d['clocks'])
for x in d.get('rows',{}).get('rows',[]):
    if x['kind']=='HSZP_ND': print(x['row'], x['api_ms'], x['kernel_ms'], x['frac'], x['kernels_us'])
P
