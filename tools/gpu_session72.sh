cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python tools/time_kkt.py 5 2>&1 | head -1
timeout 300 python tools/time_fastdiag.py 5 2>&1 | grep -i "apply" | head -3
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -k "golden or control or kkt or cfg5 or guard or timedep or determin" > gpurun_out/g72_tests.log 2>&1; tail -2 gpurun_out/g72_tests.log
