cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf -k "density or force" > gpurun_out/pytest_force.log 2>&1
echo "pytest exit $?"
timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench c3 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force_c -s 1 -c 1 -o gpurun_out/prof_force python bench.py --workload c3 --steps 5 --warmup 1 > gpurun_out/ncu_force.log 2>&1
echo "ncu exit $?"
