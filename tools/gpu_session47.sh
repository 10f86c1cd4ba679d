cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python tools/time_kkt.py 5 > gpurun_out/g47_kkt.log 2>&1; tail -3 gpurun_out/g47_kkt.log
timeout 300 python tools/time_matvec_ld.py 4 > gpurun_out/g47_ld.log 2>&1; tail -3 gpurun_out/g47_ld.log
timeout 600 python -m pytest tests -x -q -m gpu --timeout 300 -k "kkt or control or golden or guard" > gpurun_out/g47_tests.log 2>&1; tail -3 gpurun_out/g47_tests.log
