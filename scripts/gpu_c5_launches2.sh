# per-kernel durations of one C5 step in the middle of the run (after the initial sort)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -s 60 -c 40 --csv --log-file gpurun_out/c5_launches2.csv python bench.py --workload c5 --no-cpu --steps 4 --warmup 2 > gpurun_out/c5l2.log 2>&1
echo "c5 launches $?"
