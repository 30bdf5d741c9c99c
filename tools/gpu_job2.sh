# tuning job: parity tests, cell-kernel variant sweep, bench, ncu of the cell kernel
set -x
TAG=${TAG:-run}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
for v in "" _m2 _m4 _v12m4 _v12m5; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu${v}.so timeout 300 python tools/cellbench.py >> gpurun_out/${TAG}_cellbench.log 2>&1
done
timeout 300 python tools/cellbench.py --group >> gpurun_out/${TAG}_cellbench.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 300 python tools/cellbench.py > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells_t -s 3 -c 1 -o gpurun_out/${TAG}_prof_dm python tools/cellbench.py > gpurun_out/${TAG}_ncu_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells_t -s 14 -c 1 -o gpurun_out/${TAG}_prof_cvd python tools/cellbench.py >> gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
