mkdir -p gpurun_out/final
python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/final/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/final/bench.log | cut -c1-300
bash tools/launches.sh c4_16_final --views 16
bash tools/prof_kernel.sh r02c_raster_persist raster_persist 24 1 --views 16
bash tools/prof_kernel.sh r02c_tile_binning "ts_scatter|tile_sort" 50 2 --views 16
