mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/final/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/final/bench.log | cut -c1-300
for c in c1 c2 c3; do python bench.py --config $c --no-query > gpurun_out/final/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
bash tools/launches.sh c4_16_r02d --views 16
bash tools/prof_kernel.sh r02d_tile_binning "ts_scatter|tile_sort" 50 2 --views 16
