# variant sweep + diagnostics: parity tests (default build), cellbench variants, strip phase times, config sweep
set -x
TAG=${TAG:-run}
VARIANTS=${VARIANTS:-""}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
for v in "" $VARIANTS; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu${v}.so timeout 300 python tools/cellbench.py >> gpurun_out/${TAG}_cellbench.log 2>&1
done
timeout 300 python tools/strip_phase_times.py > gpurun_out/${TAG}_strip_phases.log 2>&1
timeout 900 python tools/config_sweep.py 1 2 3 4 5 > gpurun_out/${TAG}_config_sweep.log 2>&1
echo done
