# round-2 evidence (no tests): config sweep, bench launch list, ncu --set full of the top kernels
set -x
TAG=${TAG:-round2}
python -m paper_2309_13824_b200.build >/dev/null 2>&1
timeout 1200 python tools/config_sweep.py 1 2 3 4 5 > gpurun_out/${TAG}_config_sweep.jsonl 2> gpurun_out/${TAG}_config_sweep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-cfg5 --no-graph > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cells_t|k_output" -s 8 -c 5 -o gpurun_out/${TAG}_prof python tools/prof_iter.py --cfg 3 --warm 8 --warm-mode dm --modes dm cvd > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
