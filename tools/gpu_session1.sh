set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
python -m pytest tests/test_gpu_solves_full.py tests/test_gpu_configs.py -q -m gpu -x -k "cfg3_full_hgs or pinned or determin or cfg4_full" > gpurun_out/g1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g1_tests.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/g1_sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/g1_sanitize_$tool.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv -c 2 -o gpurun_out/g1_trsv_w330 python tools/prof_tri.py 5 -1 > gpurun_out/g1_ncu_trsv330.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv -c 2 -o gpurun_out/g1_trsv_w1 python tools/prof_tri.py 5 0 > gpurun_out/g1_ncu_trsv1.log 2>&1
ls -la gpurun_out
