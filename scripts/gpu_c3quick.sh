# quick C3 density/force timing + cell parity subset
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cells" > gpurun_out/q_parity.log 2>&1
echo "parity exit $?"; tail -2 gpurun_out/q_parity.log
timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 > gpurun_out/q_c3.json 2> gpurun_out/q_c3.err
python - <<'P'
import json
d = json.load(open("gpurun_out/q_c3.json"))
k = d["kernels"]
print(json.dumps({n: {kk: round(v, 4) for kk, v in r.items() if kk.endswith("_ms")} for n, r in k.items()}))
P
