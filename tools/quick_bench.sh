# quick timing only: the config-5 step and the config-4 rows of one kind ($1, default all)
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact > gpurun_out/qb_bench.log 2>&1; echo "bench rc=$?"
python - <<P
import json
l=[x for x in open('gpurun_out/qb_bench.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('step', d['ms_per_step'], 'frac', r['frac'], {k:v.get('ms_per_step') for k,v in r.get('kernels',{}).items()}, d['clocks'])
for x in d.get('rows',{}).get('rows',[]):
    if "${1:-}" in x['kind']: print(x['kind'], x['row'], x['api_ms'], x['kernel_ms'], x['frac'], x['kernels_us'])
P
