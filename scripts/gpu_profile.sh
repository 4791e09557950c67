# one ncu --set full capture per key kernel (1 GPU, short commands)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:k_gather_warp -s 5 -c 1 -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_gather.log 2>&1
echo "gather $?" >> gpurun_out/status.txt
timeout 900 $NCU -k regex:k_pairs_r -s 2 -c 1 -o gpurun_out/prof_pairs python bench.py --workload c3 --steps 5 --warmup 1 > gpurun_out/ncu_pairs.log 2>&1
echo "pairs $?" >> gpurun_out/status.txt
echo "tile $?" >> gpurun_out/status.txt
timeout 900 $NCU -k regex:k_update_soa -s 2 -c 2 -o gpurun_out/prof_update_soa python bench.py --workload c5 --c5-n 16777216 --steps 2 --warmup 1 > gpurun_out/ncu_soa.log 2>&1
echo "soa $?" >> gpurun_out/status.txt
timeout 900 $NCU -k regex:k_pack -s 1 -c 1 -o gpurun_out/prof_pack python bench.py --workload c5 --c5-n 16777216 --steps 2 --warmup 1 > gpurun_out/ncu_pack.log 2>&1
echo "pack $?" >> gpurun_out/status.txt
