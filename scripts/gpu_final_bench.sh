# final bench lines at the head (default, bf16, reference arm) and the C3 ncu metrics of the pair kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/prof
timeout 900 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench $?"
timeout 600 python bench.py --prec bf16 --no-cpu --no-extras > gpurun_out/r02_bench_c2_bf16.json 2>/dev/null; echo "bf16 $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02_bench_reference_arm.json 2>/dev/null; echo "ref $?"
bash scripts/gpu_prof_c3_final.sh
