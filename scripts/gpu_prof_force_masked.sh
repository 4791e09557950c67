# ncu of the masked force of one (smaller) C5 step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_force_masked" -s 1 -c 1 -o gpurun_out/force_masked python bench.py --workload c5 --c5-n 16777216 --no-cpu --steps 2 --warmup 1 > gpurun_out/ncu_fm.log 2>&1
echo "fm $?"; tail -3 gpurun_out/ncu_fm.log
