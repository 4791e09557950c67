cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s -C oracle > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
for w in c1 c3 c5; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "bench $w exit $?" >> gpurun_out/status.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c5.csv python bench.py --workload c5 --c5-n 16777216 --steps 2 --warmup 1 > gpurun_out/launches_c5.log 2>&1
echo "ncu c5 exit $?" >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 2 -c 1 -o gpurun_out/prof_pairs python bench.py --workload c3 --steps 5 --warmup 1 > gpurun_out/ncu_pairs.log 2>&1
echo "ncu pairs exit $?" >> gpurun_out/status.txt
