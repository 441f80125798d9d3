# A/B of the stored z scan (HSZG_CS_V: 4 = four columns per thread, unset = two for small planes); tests first
mkdir -p gpurun_out
python -m pytest tests/test_gpu_api.py tests/test_gpu_configs.py tests/test_gpu_golden.py tests/test_gpu_streaming.py tests/test_gpu_stencil.py tests/test_gpu_acceptance.py -x -q -m gpu > gpurun_out/csv_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/csv_tests.log
for v in 4 0; do
HSZG_CS_V=$v python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact > gpurun_out/csv_$v.log 2>&1
python - <<P
import json
l=[x for x in open('gpurun_out/csv_$v.log') if x.startswith('{')]
d=json.loads(l[-1])
for x in d.get('rows',{}).get('rows',[]):
    if x['kind']=='HSZP_ND' and any(s in x['row'] for s in ('A3','A13 gradient at stage 3','A7')): print('V=$v', x['row'], x['api_ms'], x['kernel_ms'], x['kernels_us'])
P
done
