# chained-iteration timing of compiled variants (A = B = the variant's default flags), 2 rounds
for r in 1 2; do
for v in "" $VARIANTS; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 600 python tools/ab_iter.py --cfg 3 4 --warm 10 --iters 6 --flags-b 0 \
    | sed "s/^/{\"lib\": \"$v\", \"r\": $r, \"d\": /; s/$/}/" >> gpurun_out/${TAG}_var.jsonl 2>>gpurun_out/${TAG}_var.err
done
done
