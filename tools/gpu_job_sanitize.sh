# compute-sanitizer memcheck on small GPU parity cases (run plain first; one sanitizer tool per call)
set -x
TAG=${TAG:-run}
SEL='test_small_random_ragged or test_octagon_binding or test_thread_kernel_overflow_retry or test_points_on_bin_edges or test_errors_are_loud'
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$SEL" > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$SEL" > gpurun_out/${TAG}_memcheck.log 2>&1; echo "memcheck exit $?" >> gpurun_out/${TAG}_memcheck.log
echo done
