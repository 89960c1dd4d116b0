# A/B timing of library builds: tools/ab.sh <tag> "<bench args>" <lib dir>... ("main" = the in-tree build)
# prints one line per (round, variant): value views/s
tag=$1; args=$2; shift 2
mkdir -p gpurun_out/ab
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=""; else lib="$v/libsemsplat_b200.so"; fi
    SS_LIB_PATH=$lib python bench.py $args --no-query --no-cpu-baseline --no-e2e > gpurun_out/ab/${tag}_${round}_$(basename $v).log 2>&1
    python - "$v" "$round" gpurun_out/ab/${tag}_${round}_$(basename $v).log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    k = d.get("kernels", {})
    print(f"{sys.argv[2]} {sys.argv[1]:12s} {d['value']:9.1f} views/s  raster {k.get('raster',{}).get('ms_per_step',0):8.2f} ms  bin {k.get('bin',{}).get('ms_per_step',0):8.2f}  contract {k.get('contract',{}).get('ms_per_step',0):8.2f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e, open(sys.argv[3]).read()[-600:])
PY
  done
done
