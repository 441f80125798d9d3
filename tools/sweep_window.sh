mkdir -p gpurun_out
for cfg in "64 256" "16 64" "16 32" "8 32" "32 64" "32 128"; do set -- $cfg
python bench.py --steps 10 --warmup 3 --window $1 --band-rows $2 --no-e2e --no-cpu --no-parity --no-exact --rows > gpurun_out/sw_$1_$2.log 2>&1
python - <<P
import json
l=[x for x in open('gpurun_out/sw_$1_$2.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); r=d['roofline']
    print('W=$1 BR=$2', d['ms_per_step'], r['frac'], {k:v.get('ms_per_step') for k,v in r.get('kernels',{}).items()})
else: print('W=$1 BR=$2 FAILED')
P
done
