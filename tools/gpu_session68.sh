cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gather_paths.py -x -q -m gpu > gpurun_out/g68_tests.log 2>&1; tail -15 gpurun_out/g68_tests.log
