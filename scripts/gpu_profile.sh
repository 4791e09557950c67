# One ncu --set full capture per key kernel plus the headline launch list (1 GPU, short commands).
# Summaries: python scripts/summarize_ncu.py gpurun_out/prof_<k>.ncu-rep profiles/r01_<k>_ncu_summary.txt "<header>"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/launches.log 2>&1
echo "launches $?"
timeout 900 $NCU -k regex:k_gather_multi -s 5 -c 1 -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_gather.log 2>&1
echo "gather $?"
timeout 900 $NCU -k regex:k_scatter_tile -s 3 -c 1 -o gpurun_out/prof_scatter python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_scatter.log 2>&1
echo "scatter $?"
timeout 900 $NCU -k regex:k_gather_multi -s 3 -c 1 -o gpurun_out/prof_gather_multi python scripts/probe_gather_one.py all > gpurun_out/ncu_gmulti.log 2>&1
echo "gather_multi $?"
timeout 900 $NCU -k regex:k_pairs_c -s 2 -c 1 -o gpurun_out/prof_pairs python bench.py --workload c3 --steps 5 --warmup 1 > gpurun_out/ncu_pairs.log 2>&1
echo "pairs $?"
timeout 900 $NCU -k regex:k_force_c -s 1 -c 1 -o gpurun_out/prof_force python bench.py --workload c3 --steps 5 --warmup 1 > gpurun_out/ncu_force.log 2>&1
echo "force $?"
timeout 900 $NCU -k regex:k_update_soa -s 2 -c 2 -o gpurun_out/prof_update_soa python bench.py --workload c5 --c5-n 16777216 --steps 2 --warmup 1 > gpurun_out/ncu_soa.log 2>&1
echo "soa $?"
timeout 900 $NCU -k regex:k_update_rec -s 6 -c 2 -o gpurun_out/prof_update_rec python bench.py --workload c1 --steps 3 --warmup 3 > gpurun_out/ncu_rec.log 2>&1
echo "rec $?"
