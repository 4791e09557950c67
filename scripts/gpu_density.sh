# density A/B: parity tests, then C3 bench per pair-kernel variant / refine
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf -k "density" > gpurun_out/pytest_density.log 2>&1
echo "pytest exit $?"
for cfg in "0 2" "1 2" "1 3" "1 4"; do
  set -- $cfg
  SFB_PAIRS=$1 timeout 600 python bench.py --workload c3 --refine $2 --steps 20 --warmup 3 > gpurun_out/bench_c3_v$1_r$2.json 2> gpurun_out/bench_c3_v$1_r$2.err
  echo "bench c3 v$1 r$2 exit $?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 2 -c 1 -o gpurun_out/prof_pairs_c python bench.py --workload c3 --steps 5 --warmup 1 > gpurun_out/ncu_pairs.log 2>&1
echo "ncu exit $?"
