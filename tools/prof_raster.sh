mkdir -p gpurun_out/r2
CMD="python bench.py --steps 1 --warmup 1 --views 6 --no-query --no-cpu-baseline --no-e2e --lanes 1"
$CMD > gpurun_out/r2/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:raster_staged -s 3 -c 1 -o gpurun_out/r2/staged $CMD > gpurun_out/r2/ncu.log 2>&1
echo rc=$?
tail -3 gpurun_out/r2/ncu.log
