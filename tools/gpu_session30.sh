cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./build_variants/dfma_lat > gpurun_out/g30_dfma_lat.log 2>&1
timeout 600 python tools/s9_trace.py > gpurun_out/g30_s9trace.log 2>&1
timeout 600 python tools/time_matvec.py 4 probe > gpurun_out/g30_matvec.log 2>&1
cat gpurun_out/g30_dfma_lat.log gpurun_out/g30_s9trace.log gpurun_out/g30_matvec.log
