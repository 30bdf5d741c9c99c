python -m paper_2309_13824_b200.build > /dev/null 2>&1
timeout 900 python tools/ab_iter.py --cfg 3 4 --warm 10 --iters 8 --flags-b 16 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
