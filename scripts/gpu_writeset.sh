# run_host mode 4 (whole records in, write set back in place): parity at 100K and 64M, C1 / C4 timings
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_sizes.py -q -x -p no:cacheprovider -k "run_host" 2>&1 | tail -2
timeout 900 python bench.py --workload c1 --no-cpu --steps 10 --warmup 3 > gpurun_out/c1w.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/c1w.json')); print('C1 e2e', d['e2e'])"
timeout 900 python bench.py --workload c4 --no-cpu --steps 5 --warmup 2 > gpurun_out/c4w.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/c4w.json')); print('C4', d.get('best_mode'), {k: round(v['ms'],1) for k,v in d['kernels'].items()}, d['roofline'])"
