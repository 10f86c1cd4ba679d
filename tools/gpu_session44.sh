cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/time_kkt.py 5 > gpurun_out/g44_kkt.log 2>&1; tail -4 gpurun_out/g44_kkt.log
SGKKT_S9_TMA=0 timeout 300 python tools/time_kkt.py 5 > gpurun_out/g44_kkt_notma.log 2>&1; tail -4 gpurun_out/g44_kkt_notma.log
timeout 300 python tools/time_matvec.py 4 > gpurun_out/g44_mv.log 2>&1; tail -2 gpurun_out/g44_mv.log
timeout 300 python tools/time_kkt.py 2 > gpurun_out/g44_kkt2.log 2>&1; tail -4 gpurun_out/g44_kkt2.log
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/g44_tests.log 2>&1; tail -5 gpurun_out/g44_tests.log
