# round-2 final evidence: smoke, every GPU test, the bench line, config sweep, the bench's launch
# list under ncu, and one ncu --set full capture of the warm cell kernels and k_output_t
set -x
TAG=${TAG:-final}
python -m paper_2309_13824_b200.build > /dev/null 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --strips --steps 2 --warmup 3 --no-cpu-baseline --no-paper-e1 > gpurun_out/${TAG}_bench_strips.log 2>&1
timeout 1200 python tools/config_sweep.py 1 2 3 4 5 > gpurun_out/${TAG}_config_sweep.jsonl 2> gpurun_out/${TAG}_config_sweep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-cfg5 --no-paper-e1 --no-graph --no-count > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cells_t|k_output" -s 16 -c 5 -o gpurun_out/${TAG}_prof python tools/prof_iter.py --cfg 3 --warm 8 --warm-mode dm --modes dm cvd > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
