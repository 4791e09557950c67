# C3 density / force timing at binning refinement 1, 2, 3, 4 (cells of side 2h / refine, reach = refine)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3 4; do
  timeout 600 python bench.py --workload c3 --no-cpu --steps 20 --warmup 3 --refine $r > gpurun_out/refine_$r.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/refine_$r.json')); k=d['kernels']
print('refine $r', {n: round(v.get('density_ms', v.get('force_ms', 0)), 4) for n, v in k.items()}, 'bin', round(k['fp32']['bin_ms'], 4))"
done
