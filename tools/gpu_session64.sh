cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py rp1 rp2 rp3 > gpurun_out/g64_ab.log 2>&1
cat gpurun_out/g64_ab.log
