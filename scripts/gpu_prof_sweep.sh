# ncu --set full of the C3 density / force sweep kernels (reports come back in gpurun_out/ for source-level reading)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:k_pairs_c -s 2 -c 1 -o gpurun_out/pairs_w python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_pairs_w.log 2>&1
echo "pairs $?"
timeout 900 $NCU -k regex:k_force_c -s 1 -c 1 -o gpurun_out/force_w python bench.py --workload c3 --no-cpu --steps 5 --warmup 1 > gpurun_out/ncu_force_w.log 2>&1
echo "force $?"
ls -la gpurun_out/*.ncu-rep
