cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py > gpurun_out/g63_ab.log 2>&1
cat gpurun_out/g63_ab.log
