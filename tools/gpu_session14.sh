cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_tri.py 5 > gpurun_out/g14_tri.log 2>&1
timeout 600 python tools/time_kkt.py 5 > gpurun_out/g14_kkt.log 2>&1
timeout 600 python tools/time_graph.py > gpurun_out/g14_graph.log 2>&1
timeout 600 python tools/triw_trace.py 64 > gpurun_out/g14_trace64.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g14_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g14_tests.log
