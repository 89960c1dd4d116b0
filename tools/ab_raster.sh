mkdir -p gpurun_out/ab
A="--steps 3 --warmup 3 --views 300 --no-query --no-cpu-baseline --no-e2e"
for round in 1 2; do
for v in "1 6" "2 6" "2 5" "2 4" "2 3"; do
  set -- $v
  SS_RASTER_CTAS_PER_SM=$2 python bench.py $A --raster $1 > gpurun_out/ab/r_${round}_$1_$2.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/ab/r_${round}_$1_$2.log').read().strip().splitlines()[-1]); k=d['kernels']
print('$round algo $1 ctas $2', round(d['value'],1), 'raster', round(k['raster']['ms_per_step'],2), 'contract', round(k['contract']['ms_per_step'],2), 'parity', d.get('parity',{}).get('ok'))
" || tail -5 gpurun_out/ab/r_${round}_$1_$2.log
done; done
