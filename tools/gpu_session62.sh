cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py gu3 gu4 gu8 > gpurun_out/g62_ab.log 2>&1
cat gpurun_out/g62_ab.log
