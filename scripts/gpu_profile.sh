# One ncu --set full capture per key kernel plus the headline launch list (1 GPU, short commands).
# Reports stay on the box (/tmp); what comes back is small: per-kernel summaries
# (scripts/summarize_ncu.py -> gpurun_out/summ_<k>.txt) and the raw metric CSVs (gpurun_out/raw_<k>.csv).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/prof
NCU="ncu --set full --clock-control none --import-source on"
summ() {  # summ <key> <header>
  python scripts/summarize_ncu.py /tmp/prof/$1.ncu-rep gpurun_out/summ_$1.txt "ncu --set full --clock-control none (scripts/gpu_profile.sh), round 1, one B200: $2"
  ncu -i /tmp/prof/$1.ncu-rep --page raw --csv > gpurun_out/raw_$1.csv 2>/dev/null
}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/launches.log 2>&1
echo "launches $?"
timeout 900 $NCU -k regex:k_gather_xv_staged -s 5 -c 1 -o /tmp/prof/gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_gather.log 2>&1
echo "gather $?"; summ gather "C2 headline step: k_gather_xv_staged (16M records, 88-B AoS -> SoA binary16 {x,v}, drift fused)"
timeout 900 $NCU -k regex:k_scatter_tile -s 3 -c 1 -o /tmp/prof/scatter python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_scatter.log 2>&1
echo "scatter $?"; summ scatter "C2 scatter-back: k_scatter_tile (binary16 x -> f64 x lanes of the 16M-record AoS)"
timeout 900 $NCU -k regex:k_gather_multi -s 3 -c 1 -o /tmp/prof/gather_multi python scripts/probe_gather_one.py all > gpurun_out/ncu_gmulti.log 2>&1
echo "gather_multi $?"; summ gather_multi "full record -> binary16: k_gather_multi<staged> (16M records)"
timeout 900 $NCU -k regex:k_pairs_c -s 2 -c 1 -o /tmp/prof/pairs python bench.py --workload c3 --steps 5 --warmup 1 > gpurun_out/ncu_pairs.log 2>&1
echo "pairs $?"; summ pairs "C3 density: k_pairs_c<2> (4M particles, fp32, uniform-h loop)"
timeout 900 $NCU -k regex:k_force_c -s 1 -c 1 -o /tmp/prof/force python bench.py --workload c3 --steps 5 --warmup 1 > gpurun_out/ncu_force.log 2>&1
echo "force $?"; summ force "C3 force: k_force_c<2,2> (4M particles, fp32, uniform-h loop)"
timeout 900 $NCU -k regex:k_update_soa -s 2 -c 2 -o /tmp/prof/update_soa python bench.py --workload c5 --c5-n 16777216 --steps 2 --warmup 1 > gpurun_out/ncu_soa.log 2>&1
echo "soa $?"; summ update_soa "C5 kick/drift on the SoA state: k_update_soa (16M particles)"
timeout 900 $NCU -k regex:k_update_rec -c 3 -o /tmp/prof/update_rec python scripts/probe_c1_kernels.py > gpurun_out/ncu_rec.log 2>&1
echo "rec $?"; summ update_rec "C1 in place on the 88-B AoS (1M records): k_update_rec_tile launches kick, drift, kick,drift"
