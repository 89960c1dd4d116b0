# SS_OPT_SORT_PREFIX sweep over 300 c4 views: tools/ab_prefix.sh <values...>
mkdir -p gpurun_out/ab
A="--steps 3 --warmup 3 --views 300 --no-query --no-cpu-baseline --no-e2e"
for round in 1 2; do
for v in "$@"; do
  python bench.py $A --sort-prefix $v > gpurun_out/ab/pf_${round}_$v.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab/pf_${round}_$v.log').read().strip().splitlines()[-1]); k=d['kernels']
print('$round prefix $v', round(d['value'],1), 'raster', round(k['raster']['ms_per_step'],2), 'bin', round(k['bin']['ms_per_step'],2))
" || tail -5 gpurun_out/ab/pf_${round}_$v.log
done; done
