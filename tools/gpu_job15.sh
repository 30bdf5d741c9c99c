set -x
TAG=${TAG:-run}
timeout 2400 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
echo done
