set -x
TAG=${TAG:-run}
timeout 600 python bench.py --steps 2 --warmup 2 --strips --no-cpu-baseline > gpurun_out/${TAG}_bench_strips1.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_bench_strips1.log
timeout 300 python tools/strip_phase_times.py > gpurun_out/${TAG}_strip_phases.log 2>&1
echo done
