cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_tri.py 5 > gpurun_out/g15_tri.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_guard.py -q -m gpu -x -k "ptilde or triangular" > gpurun_out/g15_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g15_tests.log
timeout 600 python tools/triw_trace.py 330 > gpurun_out/g15_trace330.log 2>&1
