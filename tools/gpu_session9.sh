cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_tri.py 5 > gpurun_out/g9_tri.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_fastdiag.py -q -m gpu -x -k "ptilde or fastdiag or lead_solve" > gpurun_out/g9_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g9_tests.log
timeout 600 python tools/time_fastdiag.py 5 > gpurun_out/g9_fd_time.log 2>&1
SGKKT_FD_HALF=0 timeout 600 python tools/time_fastdiag.py 5 > gpurun_out/g9_fd_time_full.log 2>&1
