cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 400 > gpurun_out/g51_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/g51_tests.log
timeout 1200 python bench.py > gpurun_out/g51_bench.log 2> gpurun_out/g51_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --impl reference > gpurun_out/g51_ref.log 2> gpurun_out/g51_ref.err; echo "ref rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:region_gemm -c 2 -o gpurun_out/g51_region -f python tools/prof_tri_wide.py 330 > gpurun_out/g51_ncu_region.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv_wide -c 2 -o gpurun_out/g51_wide330 -f python tools/prof_tri_wide.py 330 > gpurun_out/g51_ncu_wide.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/g51_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-solve-time > gpurun_out/g51_ncu_bench.log 2>&1
tail -c 600 gpurun_out/g51_bench.log
