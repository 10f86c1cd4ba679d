cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 400 > gpurun_out/g75_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/g75_tests.log
timeout 1200 python bench.py > gpurun_out/g75_bench.log 2> gpurun_out/g75_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --impl reference > gpurun_out/g75_ref.log 2> gpurun_out/g75_ref.err; echo "ref rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g75_smoke.log 2>&1; tail -1 gpurun_out/g75_smoke.log
tail -c 200 gpurun_out/g75_bench.log
