# wall-time sweep of env/bench knobs on 300 c4 views: tools/ab_knobs.sh <tag> "<env> | <bench args>"...
tag=$1; shift
mkdir -p gpurun_out/ab
A="--steps 3 --warmup 3 --views 300 --no-query --no-cpu-baseline --no-e2e"
for round in 1 2; do
  i=0
  for spec in "$@"; do
    i=$((i+1)); envs="${spec%%|*}"; args="${spec#*|}"
    f=gpurun_out/ab/${tag}_${round}_$i.log
    env $envs python bench.py $A $args > $f 2>&1
    python - "$f" "$spec" "$round" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k = d["kernels"]
    print(sys.argv[3], f"{sys.argv[2]:40s}", round(d["value"], 1), " ".join(f"{n} {v['ms_per_step']:.1f}" for n, v in k.items()))
except Exception as e:
    print(sys.argv[3], sys.argv[2], "FAILED", open(sys.argv[1]).read()[-400:])
PY
  done
done
