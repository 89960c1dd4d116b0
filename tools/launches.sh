# per-launch device times (cold, serialised) of a short bench pass: tools/launches.sh <tag> [bench args]
tag=$1; shift
mkdir -p gpurun_out/r2
CMD="python bench.py --steps 1 --warmup 1 --no-query --no-cpu-baseline --no-e2e --lanes 1 $*"
$CMD > gpurun_out/r2/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches_$tag.csv $CMD > gpurun_out/r2/ncu_$tag.log 2>&1
echo rc=$?
