cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SGKKT_S9_DEBUG=1 timeout 900 python tools/ab_variants.py shipped:SGKKT_S9_ALT2=1 2>&1 | cut -c1-400 > gpurun_out/g32_ab.log
cat gpurun_out/g32_ab.log
