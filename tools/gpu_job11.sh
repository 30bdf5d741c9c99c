set -x
TAG=${TAG:-run}
VARIANTS=${VARIANTS:-""}
for v in "" $VARIANTS; do
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu${v}.so timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/${TAG}_benchvar.log 2>&1
done
echo done
