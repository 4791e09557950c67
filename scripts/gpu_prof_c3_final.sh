# ncu --set full of the C3 pair kernels at the head: density (two homes per thread), the standalone force, and the
# masked force after a density that marked its pairs (block API step in bench c3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/prof
NCU="ncu --set full --clock-control none --import-source on"
M=gpurun_out/metrics_parts.jsonl; : > $M
summ() {
  python scripts/summarize_ncu.py /tmp/prof/$1.ncu-rep gpurun_out/r02_$1_ncu_summary.txt "ncu --set full --clock-control none (scripts/gpu_prof_c3_final.sh), round 2, one B200: $2"
  python scripts/ncu_metrics.py /tmp/prof/$1.ncu-rep $1 $3 >> $M
}
timeout 900 $NCU -k regex:k_pairs_c -s 2 -c 1 -o /tmp/prof/pairs_c3_fp32 python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_p.log 2>&1
echo "pairs $?"; summ pairs_c3_fp32 "C3 density: k_pairs_c<2> (4M, fp32, uniform h, two homes per thread, FFMA2, 48 registers)" k_pairs_c
timeout 900 $NCU -k regex:k_force_c -s 1 -c 1 -o /tmp/prof/force_c3_fp32 python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_f.log 2>&1
echo "force $?"; summ force_c3_fp32 "C3 standalone force: k_force_c<2,2> (4M, fp32, uniform-h window sweep)" k_force_c
timeout 900 $NCU -k regex:k_force_masked -s 1 -c 1 -o /tmp/prof/force_masked_c3_fp32 python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_fm.log 2>&1
echo "masked $?"; summ force_masked_c3_fp32 "C3 masked force: k_force_masked<2> after k_pairs_c wrote the window masks (4M, fp32)" k_force_masked
