cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g11_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g11_tests.log
timeout 600 python tools/triw_trace.py 64 > gpurun_out/g11_trace64.log 2>&1
timeout 600 python tools/triw_trace.py 330 > gpurun_out/g11_trace330.log 2>&1
