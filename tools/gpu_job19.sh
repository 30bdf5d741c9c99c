# quick A/B job: CVD parity tests, cellbench, bench
set -x
TAG=${TAG:-run}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "adaptive_full_size or both_cell_kernels or standalone or determinism" > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 300 python tools/cellbench.py > gpurun_out/${TAG}_cellbench.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
echo done
