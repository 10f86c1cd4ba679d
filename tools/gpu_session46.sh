cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 400 > gpurun_out/g46_tests.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/g46_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil9_tma -s 2 -c 1 -o gpurun_out/g46_tma_cfg4 -f python tools/prof_matvec.py 4 3 > gpurun_out/g46_ncu1.log 2>&1; tail -2 gpurun_out/g46_ncu1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil9_tma -s 2 -c 1 -o gpurun_out/g46_tma_kkt5 -f python tools/time_kkt.py 5 > gpurun_out/g46_ncu2.log 2>&1; tail -2 gpurun_out/g46_ncu2.log
