python -m paper_2309_13824_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1 or adaptive or determinism or graph or cfg5" > gpurun_out/d_tests.log 2>&1; echo "exit $?" >> gpurun_out/d_tests.log
VARIANTS="_nodefer" TAG=defer bash tools/gpu_job_ab3.sh
