cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SGKKT_S9_ALT2=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil9_kernel -s 2 -c 1 -o gpurun_out/g33_alt2 -f python tools/prof_matvec.py 4 3 > gpurun_out/g33_ncu.log 2>&1
tail -3 gpurun_out/g33_ncu.log
