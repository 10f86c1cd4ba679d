cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/time_tri.py 5 > gpurun_out/g48_tri_panel.log 2>&1; echo rc=$?; tail -9 gpurun_out/g48_tri_panel.log
SGKKT_TRIW_PANEL=0 timeout 600 python tools/time_tri.py 5 > gpurun_out/g48_tri_seg.log 2>&1; echo rc=$?; tail -4 gpurun_out/g48_tri_seg.log
