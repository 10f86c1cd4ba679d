cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 800 python tools/ab_variants.py shipped:SGKKT_S9_TMA=1 p_nocoef:SGKKT_S9_TMA=1 p_nov:SGKKT_S9_TMA=1 p_nosts:SGKKT_S9_TMA=1 p_all3:SGKKT_S9_TMA=1 p_gu8:SGKKT_S9_TMA=1 > gpurun_out/g42_ab.log 2>&1
cat gpurun_out/g42_ab.log
