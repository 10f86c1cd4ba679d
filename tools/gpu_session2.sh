set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/ab_matvec.py 4 > gpurun_out/g2_ab.log 2>&1
python -m pytest tests/test_gpu_solves_full.py tests/test_gpu_configs.py tests/test_gpu_golden.py tests/test_sharded.py -q -m gpu -x -k "not cfg5_full and not cfg3_full" > gpurun_out/g2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g2_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil9_grid -c 1 -o gpurun_out/g2_grid python tools/ab_matvec.py 4 > gpurun_out/g2_ncu.log 2>&1
