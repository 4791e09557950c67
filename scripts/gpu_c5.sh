cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in c3 c5 c4; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "bench $w exit $?" >> gpurun_out/status.txt
done
timeout 600 python bench.py --prec bf16 > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
echo "bench bf16 exit $?" >> gpurun_out/status.txt
