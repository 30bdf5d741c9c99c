set -x
TAG=${TAG:-run}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 900 python tools/config_sweep.py 2 3 4 5 > gpurun_out/${TAG}_config_sweep.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
echo done
