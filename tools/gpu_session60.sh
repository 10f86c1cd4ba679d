cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py ldc > gpurun_out/g60_ab.log 2>&1
cat gpurun_out/g60_ab.log
