# full GPU test suite + C3 / C5 / C5-full bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
timeout 900 python bench.py --workload c3 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench c3 exit $?"
timeout 900 python bench.py --workload c5 --steps 5 --warmup 2 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "bench c5 exit $?"
timeout 900 python bench.py --workload c5 --steps 5 --warmup 2 > gpurun_out/bench_c5_full.json 2> gpurun_out/bench_c5_full.err
echo "bench c5 full exit $?"
