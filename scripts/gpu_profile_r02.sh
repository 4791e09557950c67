# Round-2 evidence: the headline launch list and one `ncu --set full` per key kernel (1 GPU, short
# commands).  Reports stay on the box; summaries (scripts/summarize_ncu.py) and key metrics
# (scripts/ncu_metrics.py -> kernel_metrics.json) come back in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/prof
NCU="ncu --set full --clock-control none --import-source on"
M=gpurun_out/metrics_parts.jsonl; : > $M
summ() {  # summ <key> <header>
  python scripts/summarize_ncu.py /tmp/prof/$1.ncu-rep gpurun_out/r02_$1_ncu_summary.txt "ncu --set full --clock-control none (scripts/gpu_profile_r02.sh), round 2, one B200: $2"
  python scripts/ncu_metrics.py /tmp/prof/$1.ncu-rep $1 >> $M
}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/launches.log 2>&1
echo "launches $?"
timeout 900 $NCU -k regex:k_gather_xv_staged -s 5 -c 1 -o /tmp/prof/gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_gather.log 2>&1
echo "gather $?"; summ gather "C2 headline step: k_gather_xv_staged (16M records, 88-B AoS -> SoA binary16 {x,v}, drift fused)"
timeout 900 $NCU -k regex:k_scatter_tile -s 3 -c 1 -o /tmp/prof/scatter python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_scatter.log 2>&1
echo "scatter $?"; summ scatter "C2 scatter-back: k_scatter_tile (binary16 x -> f64 x lanes of the 16M-record AoS)"
timeout 900 $NCU -k regex:k_pairs_c -s 2 -c 1 -o /tmp/prof/pairs_c3_fp32 python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_pairs.log 2>&1
echo "pairs $?"; summ pairs_c3_fp32 "C3 density: k_pairs_c<2> (4M particles, fp32, uniform-h loop, one float4 per candidate)"
timeout 900 $NCU -k regex:k_force_c -s 1 -c 1 -o /tmp/prof/force_c3_fp32 python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_force.log 2>&1
echo "force $?"; summ force_c3_fp32 "C3 force: k_force_c<2,2> (4M particles, fp32, uniform-h loop)"
timeout 900 $NCU -k regex:k_update_rec_tile -c 3 -o /tmp/prof/update_rec python scripts/probe_c1_kernels.py > gpurun_out/ncu_rec.log 2>&1
echo "rec $?"; summ update_rec "C1 in place on the 88-B AoS (1M records): k_update_rec_tile launches kick, drift, kick,drift"
timeout 1200 $NCU -k regex:"k_pairs_c|k_force_c|k_cell_rank|k_pack" -s 12 -c 5 -o /tmp/prof/c5 python bench.py --workload c5 --no-cpu --steps 2 --warmup 1 > gpurun_out/ncu_c5.log 2>&1
echo "c5 $?"; python scripts/summarize_ncu.py /tmp/prof/c5.ncu-rep gpurun_out/r02_c5_ncu_summary.txt "ncu --set full, round 2: one C5 step (128M, N=1): binning, pack, k_pairs_c, k_force_c"
