# Round-2 evidence on one B200: the GPU test suite, smoke, the default bench line (C2 + every extra), the bf16
# headline, the reference arm, and compute-sanitizer over the shard / edge-case tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nvidia-smi; nproc; lscpu | head -20; free -g) > gpurun_out/r02_box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 600 > gpurun_out/r02_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench $?"
timeout 600 python bench.py --prec bf16 --no-cpu --no-extras > gpurun_out/r02_bench_c2_bf16.json 2>/dev/null; echo "bf16 $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02_bench_reference_arm.json 2>/dev/null; echo "ref $?"
SAN="compute-sanitizer --error-exitcode 9"
( for tool in memcheck racecheck synccheck; do
    echo "== $tool: shard across processes is not run under the sanitizer (CUDA IPC between sanitized processes); single-rank shard + edge cases"
    timeout 900 $SAN --tool $tool python -m pytest -q -p no:cacheprovider tests/test_gpu_sharded.py -k "single_rank or uniform" tests/test_gpu_parity.py -k "ragged or zero_records or wide_records or shifted or force_large or single_rank or uniform" 2>&1 | tail -4
    echo "exit $?"
  done ) > gpurun_out/r02_sanitizer.txt 2>&1
echo "sanitizer done"; grep -E "ERROR SUMMARY|passed|failed|exit" gpurun_out/r02_sanitizer.txt | head -12
