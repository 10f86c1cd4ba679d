cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/triw_trace.py 64 > gpurun_out/g7_trace64.log 2>&1
timeout 600 python tools/triw_trace.py 330 > gpurun_out/g7_trace330.log 2>&1
