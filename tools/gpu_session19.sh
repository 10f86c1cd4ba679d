cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/ab_matvec.py 4 > gpurun_out/g19_ab.log 2>&1
SGKKT_GRID9=1 timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_guard.py tests/test_gpu_solves_full.py -q -m gpu -x -k "cfg4 or pinned or coupling" > gpurun_out/g19_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g19_tests.log
cat gpurun_out/g19_ab.log; tail -3 gpurun_out/g19_tests.log
