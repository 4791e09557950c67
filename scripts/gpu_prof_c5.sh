# ncu --set full of one C5 step's pair kernels (density with window masks, masked force)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_pairs_c|k_force_masked|k_force_c" -s 4 -c 2 -o gpurun_out/c5_pairs python bench.py --workload c5 --no-cpu --steps 2 --warmup 1 > gpurun_out/ncu_c5p.log 2>&1
echo "c5 $?"
