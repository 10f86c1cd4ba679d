cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 400 > gpurun_out/g73_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/g73_tests.log
timeout 1200 python bench.py > gpurun_out/g73_bench.log 2> gpurun_out/g73_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --impl reference > gpurun_out/g73_ref.log 2> gpurun_out/g73_ref.err; echo "ref rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g73_smoke.log 2>&1; tail -1 gpurun_out/g73_smoke.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/g73_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-solve-time > gpurun_out/g73_ncu_bench.log 2>&1
tail -c 200 gpurun_out/g73_bench.log
