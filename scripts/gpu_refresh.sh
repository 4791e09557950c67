# Refresh every bench line kept under profiles/ (one B200), plus tests and smoke.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nvidia-smi; nproc; lscpu | head -20) > gpurun_out/box.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r01_bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 $?"
timeout 900 python bench.py --prec bf16 --no-cpu > gpurun_out/r01_bench_c2_bf16.json 2>/dev/null; echo "c2 bf16 $?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r01_bench_reference_arm.json 2>/dev/null; echo "ref $?"
for w in c1 c3 c4 c5; do
  timeout 1200 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/r01_bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w $?"
done
timeout 1200 python bench.py --workload c5 --steps 5 --warmup 2 > gpurun_out/r01_bench_c5_full.json 2>/dev/null; echo "c5 full $?"
