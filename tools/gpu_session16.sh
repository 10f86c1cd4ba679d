cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/ab_matvec.py 4 > gpurun_out/g16_ab.log 2>&1
cat gpurun_out/g16_ab.log
