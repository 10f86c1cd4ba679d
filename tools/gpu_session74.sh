cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python tools/time_kkt.py 5 2>&1 | head -1
timeout 300 python tools/time_fastdiag.py 5 2>&1 | grep -i "hgsoc\[fastdiag\] apply\|blockdiag\[fastdiag\] apply" | head -3
timeout 200 python tools/time_matvec.py 2 2>&1 | tail -1 | cut -c1-50
