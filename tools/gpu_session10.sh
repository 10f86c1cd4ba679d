cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fastdiag.py -q -m gpu -x > gpurun_out/g10_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g10_tests.log
timeout 600 python tools/time_fastdiag.py 5 > gpurun_out/g10_fd_time.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_probe tools/fp64_probe.cu > gpurun_out/g10_probe_build.log 2>&1 && /tmp/fp64_probe > gpurun_out/g10_fp64_probe.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fdh_ -c 3 --launch-skip 30 -o gpurun_out/g10_fdh python tools/time_fastdiag.py 5 > gpurun_out/g10_ncu.log 2>&1
