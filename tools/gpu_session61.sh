cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py hint gu4 > gpurun_out/g61_ab.log 2>&1
cat gpurun_out/g61_ab.log
