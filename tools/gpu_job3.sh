# sweep job: parity tests on the default build, variant + n_opt sweep of the cell kernel, bench
set -x
TAG=${TAG:-run}
VARIANTS=${VARIANTS:-""}
NOPT=${NOPT:-3.3,6}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
for v in "" $VARIANTS; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu${v}.so timeout 300 python tools/cellbench.py --n-opt=$NOPT >> gpurun_out/${TAG}_cellbench.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log

timeout 600 python bench.py --steps 2 --warmup 3 --strips --no-cpu-baseline > gpurun_out/${TAG}_bench_strips1.log 2>&1; echo "strips bench exit $?" >> gpurun_out/${TAG}_bench_strips1.log
echo done
