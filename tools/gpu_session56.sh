cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_variants.py shipped:SGKKT_GRID9=1 shipped:SGKKT_GRID9=1,SGKKT_GRID_TMA=0 > gpurun_out/g56_ab.log 2>&1
cat gpurun_out/g56_ab.log
SGKKT_GRID9=1 timeout 600 python -m pytest tests -x -q -m gpu --timeout 300 -k "grid or cfg4 or guard or golden or sharded or pinned" > gpurun_out/g56_tests.log 2>&1; tail -3 gpurun_out/g56_tests.log
