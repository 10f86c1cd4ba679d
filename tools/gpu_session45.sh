cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SGKKT_S9_DEBUG=1 timeout 120 python tools/time_kkt.py 5 > gpurun_out/g45_kkt.log 2>&1; echo rc=$?; grep -v "^stencil9_tma" gpurun_out/g45_kkt.log | tail -4; grep "^stencil9_tma" gpurun_out/g45_kkt.log | sort | uniq -c
SGKKT_S9_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_configs.py -x -q -m gpu -k "test_control_hgsoc_fgmres_and_minres" > gpurun_out/g45_t9.log 2>&1; echo rc=$?; grep -v "^stencil9_tma" gpurun_out/g45_t9.log | tail -5; grep "^stencil9_tma" gpurun_out/g45_t9.log | sort | uniq -c | tail; tail -3 gpurun_out/g45_t9.log
