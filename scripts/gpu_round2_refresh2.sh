# Round-2 evidence after the window-mask force: full GPU suite, smoke, ncu of the C5 pair kernels, default bench,
# bf16, reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/prof
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 600 > gpurun_out/r02_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke exit $?"
NCU="ncu --set full --clock-control none --import-source on"
M=gpurun_out/metrics_parts.jsonl; : > $M
timeout 1500 $NCU -k regex:"k_cell_rank|k_pack|k_pairs_c|k_force_masked" -s 12 -c 6 -o /tmp/prof/c5 python bench.py --workload c5 --no-cpu --steps 2 --warmup 1 > gpurun_out/ncu_c5.log 2>&1
echo "c5 ncu $?"; python scripts/summarize_ncu.py /tmp/prof/c5.ncu-rep gpurun_out/r02_c5_ncu_summary.txt "ncu --set full, round 2: one C5 step (128M, N=1): binning, pack, k_pairs_c with window masks, k_force_masked"
python scripts/ncu_metrics.py /tmp/prof/c5.ncu-rep pairs_c5 k_pairs_c >> $M
python scripts/ncu_metrics.py /tmp/prof/c5.ncu-rep force_c5 k_force_masked >> $M
timeout 900 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench $?"
timeout 600 python bench.py --prec bf16 --no-cpu --no-extras > gpurun_out/r02_bench_c2_bf16.json 2>/dev/null; echo "bf16 $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02_bench_reference_arm.json 2>/dev/null; echo "ref $?"
