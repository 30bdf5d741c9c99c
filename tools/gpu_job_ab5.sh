# A/B of compiled variants ($VARIANTS, e.g. "_pf"): parity of each variant on the GPU parity
# subset, chained-iteration timing (gpu_job_ab3.sh), and one ncu --set full capture (source
# level) of the default library's warm DistMesh and CVD cell launches
set -x
TAG=${TAG:-ab5}
python -m paper_2309_13824_b200.build > /dev/null 2>&1
for v in $VARIANTS; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q \
    -k "cfg1 or cfg2 or adaptive or both_cell or small_random or octagon or bin_edges" > gpurun_out/${TAG}_parity$v.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${TAG}_parity$v.log
done
VARIANTS="$VARIANTS" TAG=$TAG bash tools/gpu_job_ab3.sh
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cells_t" -s 8 -c 2 -o gpurun_out/${TAG}_prof python tools/prof_iter.py --cfg 3 --warm 8 --warm-mode dm --modes dm cvd > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
echo done
