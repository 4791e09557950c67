cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s -C oracle > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/status.txt
for w in c1 c5; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "bench $w exit $?" >> gpurun_out/status.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather -s 5 -c 1 -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/launches.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/status.txt
