cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py > gpurun_out/g13_bench.log 2> gpurun_out/g13_bench.err
echo "bench rc=$?" >> gpurun_out/g13_bench.err
python bench.py --impl reference > gpurun_out/g13_ref.log 2> gpurun_out/g13_ref.err
echo "ref rc=$?" >> gpurun_out/g13_ref.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil9_ws -c 1 -o gpurun_out/g13_ws python tools/time_matvec.py 4 > gpurun_out/g13_ncu_ws.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv_wide -c 2 -o gpurun_out/g13_wide330 python tools/prof_tri_wide.py 330 > gpurun_out/g13_ncu_wide.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fdh_ -c 3 --launch-skip 12 -o gpurun_out/g13_fdh python tools/time_fastdiag.py 5 > gpurun_out/g13_ncu_fdh.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/g13_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-solve-time > gpurun_out/g13_ncu_bench.log 2>&1
