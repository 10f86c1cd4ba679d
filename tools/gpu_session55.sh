cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py p_v3 > gpurun_out/g55_ab.log 2>&1
cat gpurun_out/g55_ab.log
