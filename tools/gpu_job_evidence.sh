# evidence only (no tests): config sweep, launch list of the bench, ncu --set full of the cell kernels
set -x
TAG=${TAG:-run}
timeout 900 python tools/config_sweep.py 1 2 3 4 5 > gpurun_out/${TAG}_config_sweep.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells_t -s 3 -c 1 -o gpurun_out/${TAG}_prof_dm python tools/cellbench.py > gpurun_out/${TAG}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cells_t|k_output_t" -s 17 -c 2 -o gpurun_out/${TAG}_prof_cvd python tools/cellbench.py >> gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
