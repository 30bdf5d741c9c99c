python -m paper_2309_13824_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_strips.py tests/test_gpu_next1.py -x -q > gpurun_out/t_tests.log 2>&1; echo "exit $?" >> gpurun_out/t_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-paper-e1 > gpurun_out/bg.log 2>&1
