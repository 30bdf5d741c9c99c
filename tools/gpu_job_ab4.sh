python -m paper_2309_13824_b200.build > /dev/null 2>&1
VARIANTS="$VARIANTS" TAG=$TAG bash tools/gpu_job_ab3.sh
