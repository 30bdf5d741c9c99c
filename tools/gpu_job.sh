# one gpurun job: GPU parity tests, bench (thread + group A/B), launch list and
# one ncu --set full capture of the cell kernel.  Outputs under gpurun_out/.
set -x
TAG=${TAG:-run}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 600 python bench.py --steps 2 --warmup 3 --cells group --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_group.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 300 python tools/profile_step.py 3 > gpurun_out/${TAG}_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells -s 8 -c 4 -o gpurun_out/${TAG}_prof_cells python tools/profile_step.py 3 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
