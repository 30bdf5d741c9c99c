set -x
TAG=${TAG:-run}
VARIANTS=${VARIANTS:-""}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
TRIME_LIB=paper_2309_13824_b200/libtrime_gpu_cs2.so timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests_cs2.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests_cs2.log
for v in "" $VARIANTS; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu${v}.so timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_benchvar.log 2>&1
done
echo done
