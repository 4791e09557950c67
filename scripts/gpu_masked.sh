# masked density/force parity + the C3 density-then-force measurement
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sharded.py -q -x -p no:cacheprovider -k "masked" > gpurun_out/masked.log 2>&1
echo "masked exit $?"; tail -3 gpurun_out/masked.log
timeout 600 python bench.py --workload c3 --no-cpu --steps 20 --warmup 3 > gpurun_out/c3m.json 2> gpurun_out/c3m.err
python -c "
import json; d=json.load(open('gpurun_out/c3m.json')); print(json.dumps(d['kernels'].get('step_fp32')))"
