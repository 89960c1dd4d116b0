# pipeline balance sweep over 300 c4 views: contraction CTAs x lanes
mkdir -p gpurun_out/ab
A="--steps 3 --warmup 3 --views 300 --no-query --no-cpu-baseline --no-e2e"
for round in 1 2; do
for v in ${KNOBS:-"89 5" "74 6" "60 6" "66 6" "74 5"}; do
  set -- $v
  SS_CONTRACT_CTAS=$1 python bench.py $A --lanes $2 > gpurun_out/ab/kn_${round}_$1_$2.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab/kn_${round}_$1_$2.log').read().strip().splitlines()[-1])
print('$round ctas $1 lanes $2', round(d['value'],1))
" || tail -3 gpurun_out/ab/kn_${round}_$1_$2.log
done; done
