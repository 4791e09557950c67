cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf -k "force" > gpurun_out/pytest_force.log 2>&1
echo "pytest exit $?"
for u in 1 2; do
SFB_FORCE_UNROLL=$u timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 > gpurun_out/bench_c3_u$u.json 2> gpurun_out/bench_c3_u$u.err
echo "bench c3 u$u exit $?"
done
