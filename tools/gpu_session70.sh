cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:program_kernel -s 2 -c 1 -o gpurun_out/g70_prog_cfg3 -f python tools/prof_matvec.py 3 3 > gpurun_out/g70_ncu.log 2>&1; tail -2 gpurun_out/g70_ncu.log
