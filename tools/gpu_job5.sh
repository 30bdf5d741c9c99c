# validation + profile of the cell kernel; strips bench smoke
set -x
TAG=${TAG:-run}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 300 python tools/cellbench.py > gpurun_out/${TAG}_cellbench.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 600 python bench.py --steps 2 --warmup 3 --strips --no-cpu-baseline > gpurun_out/${TAG}_bench_strips1.log 2>&1; echo "strips bench exit $?" >> gpurun_out/${TAG}_bench_strips1.log
timeout 300 python tools/cellbench.py > gpurun_out/${TAG}_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells_t -s 3 -c 1 -o gpurun_out/${TAG}_prof_dm python tools/cellbench.py > gpurun_out/${TAG}_ncu_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells_t -s 14 -c 1 -o gpurun_out/${TAG}_prof_cvd python tools/cellbench.py >> gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
