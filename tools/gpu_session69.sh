cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py sl20 sl100 > gpurun_out/g69_ab.log 2>&1
cat gpurun_out/g69_ab.log
