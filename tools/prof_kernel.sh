# ncu --set full of kernels matching a regex in a short bench pass: tools/prof_kernel.sh <tag> <regex> <skip> <count> [bench args]
tag=$1; rx=$2; skip=$3; cnt=$4; shift 4
mkdir -p gpurun_out/r2
CMD="python bench.py --steps 1 --warmup 1 --no-query --no-cpu-baseline --no-e2e --lanes 1 $*"
$CMD > gpurun_out/r2/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c $cnt -o gpurun_out/r2/$tag $CMD > gpurun_out/r2/ncu_$tag.log 2>&1
echo rc=$?
tail -2 gpurun_out/r2/ncu_$tag.log
