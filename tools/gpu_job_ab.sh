# A/B of compiled library variants against the default build with tools/cellbench.py,
# alternating order, 2 rounds.
# Build variants first, e.g. build(out=".../libtrime_gpu_x.so", defines=["TM_X=1"]), then
#   VARIANTS="_x _y" CFGS="3 4 5" TAG=r9 bash tools/gpu_job_ab.sh
TAG=${TAG:-run}
VARIANTS=${VARIANTS:-""}
CFGS=${CFGS:-"3 4"}
for r in 1 2; do
for v in "" $VARIANTS; do
  for c in $CFGS; do
    TRIME_LIB=paper_2309_13824_b200/libtrime_gpu$v.so timeout 300 python tools/cellbench.py --cfg=$c \
      >> gpurun_out/${TAG}_variants.jsonl 2>>gpurun_out/${TAG}_variants.err
  done
done
done
echo done
