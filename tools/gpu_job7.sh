# distribution study: cellbench on cfg3 / iid 1e6 / cfg5 (1.6e7), ncu of the iid DM launch; bench
set -x
TAG=${TAG:-run}
for c in 3 iid 5; do timeout 600 python tools/cellbench.py --cfg=$c >> gpurun_out/${TAG}_cellbench.log 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 300 python tools/cellbench.py --cfg=iid > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells_t -s 3 -c 1 -o gpurun_out/${TAG}_prof_iid_dm python tools/cellbench.py --cfg=iid > gpurun_out/${TAG}_ncu.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cells_t -s 3 -c 1 -o gpurun_out/${TAG}_prof_cfg3_dm python tools/cellbench.py --cfg=3 >> gpurun_out/${TAG}_ncu.log 2>&1
echo done
