# A/B of compiled cell-kernel variants (round 2) + parity of the combined variant
TAG=${TAG:-run}
TRIME_LIB=paper_2309_13824_b200/libtrime_gpu_all.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "adaptive_full_size or both_cell_kernels or small_random or near_cocircular or points_on_bin" > gpurun_out/${TAG}_all_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_all_tests.log
for r in 1 2; do
for v in "" _both _share _all; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 300 python tools/cellbench.py >> gpurun_out/${TAG}_variants.jsonl 2>>gpurun_out/${TAG}_variants.err
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 300 python tools/cellbench.py --cfg=4 >> gpurun_out/${TAG}_variants.jsonl 2>>gpurun_out/${TAG}_variants.err
done
done
echo done
