cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_tri.py 5 > gpurun_out/g5_tri.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv_wide -c 2 -o gpurun_out/g5_wide330 python tools/prof_tri_wide.py 330 > gpurun_out/g5_ncu330.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv_wide -c 2 -o gpurun_out/g5_wide64 python tools/prof_tri_wide.py 64 > gpurun_out/g5_ncu64.log 2>&1
