cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/time_tri.py 5 > gpurun_out/g53_tri.log 2>&1; echo rc=$?; tail -9 gpurun_out/g53_tri.log
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -k "tri or lu or guard or cfg5 or solves_full or golden" > gpurun_out/g53_tests.log 2>&1; tail -2 gpurun_out/g53_tests.log
