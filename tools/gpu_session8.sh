cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_tri.py 5 > gpurun_out/g8_tri.log 2>&1
timeout 600 python tools/triw_trace.py 64 > gpurun_out/g8_trace64.log 2>&1
timeout 600 python tools/triw_trace.py 330 > gpurun_out/g8_trace330.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -m gpu -x -k "ptilde" > gpurun_out/g8_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g8_tests.log
