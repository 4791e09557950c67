# Warp-cooperative density / force sweep: parity (cell tests, BASELINE sizes, shard) and C3 / C5 timings.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cell or force or density" > gpurun_out/sweep_parity.log 2>&1
echo "parity exit $?"; tail -3 gpurun_out/sweep_parity.log
timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider -k "c3 or c5 or C3 or C5 or shard or block" > gpurun_out/sweep_sizes.log 2>&1
echo "sizes exit $?"; tail -3 gpurun_out/sweep_sizes.log
timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 > gpurun_out/sweep_c3.json 2> gpurun_out/sweep_c3.err
echo "c3 $?"
python - <<'P'
import json
d = json.load(open("gpurun_out/sweep_c3.json"))
k = d.get("kernels", d.get("configs", {}).get("c3", {}).get("kernels", {}))
print(json.dumps({n: {kk: v for kk, v in r.items() if kk.endswith("_ms")} for n, r in k.items()}))
P
timeout 900 python bench.py --workload c5 --steps 3 --warmup 2 > gpurun_out/sweep_c5.json 2> gpurun_out/sweep_c5.err
echo "c5 $?"
python -c "
import json; d=json.load(open('gpurun_out/sweep_c5.json')); print(d.get('ms_per_step'), d.get('phases_ms_max_over_ranks') or d.get('phases_ms'))"
