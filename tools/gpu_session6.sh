cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fastdiag.py -q -m gpu -x > gpurun_out/g6_fd_tests.log 2>&1
echo "rc=$?" >> gpurun_out/g6_fd_tests.log
timeout 600 python tools/time_fastdiag.py 5 > gpurun_out/g6_fd_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fd_ -c 3 -o gpurun_out/g6_fd python tools/time_fastdiag.py 5 > gpurun_out/g6_ncu.log 2>&1
