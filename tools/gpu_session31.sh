cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/ab_variants.py gu4 gu8 ce gu4ce > gpurun_out/g31_ab.log 2>&1
cat gpurun_out/g31_ab.log
