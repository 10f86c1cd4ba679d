cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py shipped:SGKKT_GRID_TMA=2 > gpurun_out/g59_ab.log 2>&1
cat gpurun_out/g59_ab.log
