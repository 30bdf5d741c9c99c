set -x
TAG=${TAG:-run}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "capacity_error or cocircular or errors_are_loud" > gpurun_out/${TAG}_new_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_new_tests.log
echo done
