cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --workload c5 --steps 5 --warmup 2 > gpurun_out/c5q.json 2> gpurun_out/c5q.err
python -c "
import json; d=json.load(open('gpurun_out/c5q.json')); print(d.get('ms_per_step'), d.get('phases_ms_max_over_ranks') or d.get('phases_ms'))"
