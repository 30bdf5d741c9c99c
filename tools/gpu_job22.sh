# leaf bounding-box pruning: parity subset, cellbench A/B (box vs nobox), bench
TAG=${TAG:-run}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_strips.py -m gpu -x -q -k "adaptive_full_size or both_cell_kernels or small_random or near_cocircular or points_on_bin or cfg2 or octagon or loopback or adaptive_halo" > gpurun_out/${TAG}_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_tests.log
for r in 1 2; do
for v in "" _nobox; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 300 python tools/cellbench.py >> gpurun_out/${TAG}_variants.jsonl 2>>gpurun_out/${TAG}_variants.err
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 300 python tools/cellbench.py --cfg=4 >> gpurun_out/${TAG}_variants.jsonl 2>>gpurun_out/${TAG}_variants.err
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 300 python tools/cellbench.py --cfg=5 >> gpurun_out/${TAG}_variants.jsonl 2>>gpurun_out/${TAG}_variants.err
done
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
echo done
