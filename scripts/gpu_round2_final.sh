# Round-2 refresh after the density change: ncu --set full of C3 density / force and one C5 step (metrics for
# profiles/kernel_metrics.json), then the default bench line, bf16 and the reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/prof
NCU="ncu --set full --clock-control none --import-source on"
M=gpurun_out/metrics_parts.jsonl; : > $M
summ() {  # summ <key> <header>
  python scripts/summarize_ncu.py /tmp/prof/$1.ncu-rep gpurun_out/r02_$1_ncu_summary.txt "ncu --set full --clock-control none (scripts/gpu_round2_final.sh), round 2, one B200: $2"
  python scripts/ncu_metrics.py /tmp/prof/$1.ncu-rep $1 >> $M
}
timeout 900 $NCU -k regex:k_pairs_c -s 2 -c 1 -o /tmp/prof/pairs_c3_fp32 python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_pairs.log 2>&1
echo "pairs $?"; summ pairs_c3_fp32 "C3 density: k_pairs_c<2> (4M particles, fp32, uniform h: two homes per thread, FFMA2 pair terms)"
timeout 900 $NCU -k regex:k_force_c -s 1 -c 1 -o /tmp/prof/force_c3_fp32 python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_force.log 2>&1
echo "force $?"; summ force_c3_fp32 "C3 force: k_force_c<2,2> (4M particles, fp32, uniform-h loop)"
timeout 1200 $NCU -k regex:"k_pairs_c|k_force_c|k_cell_rank|k_pack" -s 12 -c 5 -o /tmp/prof/c5 python bench.py --workload c5 --no-cpu --steps 2 --warmup 1 > gpurun_out/ncu_c5.log 2>&1
echo "c5 $?"; python scripts/summarize_ncu.py /tmp/prof/c5.ncu-rep gpurun_out/r02_c5_ncu_summary.txt "ncu --set full, round 2: one C5 step (128M, N=1): binning, pack, k_pairs_c, k_force_c"
python scripts/ncu_metrics.py /tmp/prof/c5.ncu-rep pairs_c5 k_pairs_c >> $M
python scripts/ncu_metrics.py /tmp/prof/c5.ncu-rep force_c5 k_force_c >> $M
timeout 900 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench $?"
timeout 600 python bench.py --prec bf16 --no-cpu --no-extras > gpurun_out/r02_bench_c2_bf16.json 2>/dev/null; echo "bf16 $?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02_bench_reference_arm.json 2>/dev/null; echo "ref $?"
