# launch list (per-kernel durations) of C5 steps at N=1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 36 -c 30 --csv --log-file gpurun_out/c5_launches.csv python bench.py --workload c5 --no-cpu --steps 2 --warmup 1 > gpurun_out/c5l.log 2>&1
echo "c5 launches $?"
