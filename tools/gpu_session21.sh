cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/g21_bench.log 2> gpurun_out/g21_bench.err
echo "bench rc=$?" >> gpurun_out/g21_bench.err
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/g21_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g21_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g21_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/g21_smoke.log
