# A/B of compiled cell-kernel variants with tools/cellbench.py (alternating order, 2 rounds)
TAG=${TAG:-run}
for r in 1 2; do
for v in "" _lim _fast _both; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 300 python tools/cellbench.py >> gpurun_out/${TAG}_variants.jsonl 2>>gpurun_out/${TAG}_variants.err
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 300 python tools/cellbench.py --cfg=4 >> gpurun_out/${TAG}_variants.jsonl 2>>gpurun_out/${TAG}_variants.err
done
done
echo done
