python -m paper_2309_13824_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_strips.py -x -q > gpurun_out/t_tests.log 2>&1; echo "exit $?" >> gpurun_out/t_tests.log
