cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python tools/time_kkt.py 5 2>&1 | head -1
SGKKT_B200_LIB=$PWD/build_variants/libsgkkt_altldc.so timeout 200 python tools/time_kkt.py 5 2>&1 | head -1
timeout 300 python tools/time_fastdiag.py 5 2>&1 | grep -i "apply" | head -3
SGKKT_B200_LIB=$PWD/build_variants/libsgkkt_altldc.so timeout 300 python tools/time_fastdiag.py 5 2>&1 | grep -i "apply" | head -3
