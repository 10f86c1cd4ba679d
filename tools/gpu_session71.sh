cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/time_matvec.py 3 2>&1 | tail -1 | cut -c1-60
timeout 600 python -m pytest tests -x -q -m gpu --timeout 300 -k "cfg3 or guard or golden or program or capi" > gpurun_out/g71_tests.log 2>&1; tail -2 gpurun_out/g71_tests.log
