# A/B of the stage-3 HSZP_ND band height (HSZG_RECON_BR) on the config-4 rows
mkdir -p gpurun_out
for br in 0 256 128; do
HSZG_RECON_BR=$br python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-exact > gpurun_out/br_$br.log 2>&1
python - <<P
import json
l=[x for x in open('gpurun_out/br_$br.log') if x.startswith('{')]
d=json.loads(l[-1])
for x in d.get('rows',{}).get('rows',[]):
    if x['kind']=='HSZP_ND' and any(s in x['row'] for s in ('A3','N1 variance at stage 3','A13 gradient at stage 3','N2')): print('BR=$br', x['row'], x['api_ms'], x['kernel_ms'], x['kernels_us'])
P
done
