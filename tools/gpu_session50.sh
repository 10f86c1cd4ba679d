cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/time_tri.py 5 > gpurun_out/g50_tri.log 2>&1; echo rc=$?; tail -9 gpurun_out/g50_tri.log
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -k "tri or lu or guard or solves_full or cfg5" > gpurun_out/g50_tests.log 2>&1; tail -3 gpurun_out/g50_tests.log
