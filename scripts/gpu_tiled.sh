cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf -k "density or force or shard or outside" > gpurun_out/pytest_tiled.log 2>&1
echo "pytest exit $?"
for t in 0 1; do
SFB_TILED=$t timeout 900 python bench.py --workload c5 --c5-full --steps 3 --warmup 1 > gpurun_out/bench_c5f_t$t.json 2> gpurun_out/bench_c5f_t$t.err
SFB_TILED=$t timeout 900 python bench.py --workload c3 --steps 10 --warmup 2 > gpurun_out/bench_c3_t$t.json 2> gpurun_out/bench_c3_t$t.err
echo "bench t$t exit $?"
done
