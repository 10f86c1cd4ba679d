cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/time_tri.py 5 > gpurun_out/g52_tri.log 2>&1; echo rc=$?; tail -6 gpurun_out/g52_tri.log
SGKKT_TRIW_TILE_ENTRIES=512 SGKKT_TRIW_TILE_SEGS=16 timeout 300 python tools/time_tri.py 5 > gpurun_out/g52_tri_t512.log 2>&1; echo rc=$?; tail -6 gpurun_out/g52_tri_t512.log
timeout 600 python -m pytest tests -x -q -m gpu --timeout 300 -k "tri or lu or guard or cfg5" > gpurun_out/g52_tests.log 2>&1; tail -2 gpurun_out/g52_tests.log
