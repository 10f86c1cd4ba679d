cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_tri.py 5 > gpurun_out/g22_tri.log 2>&1
SGKKT_B200_LIB=$PWD/build_variants/libsgkkt_allfence.so timeout 900 python tools/time_tri.py 5 > gpurun_out/g22_tri_allfence.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_guard.py -q -m gpu -x -k "ptilde or triangular" > gpurun_out/g22_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g22_tests.log
grep -h "width\|apply" gpurun_out/g22_tri.log gpurun_out/g22_tri_allfence.log; tail -2 gpurun_out/g22_tests.log
