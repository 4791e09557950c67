# sweep the gather's TMA ring depth and warps/SM on the C2 headline
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for st in 3 4 6 8; do for w in 8 12 16; do
  r=$(SFB_GATHER_STAGES=$st SFB_GATHER_WARPS=$w timeout 300 python bench.py --no-e2e --no-cpu --steps 100 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "stages=$st warps=$w $r" >> gpurun_out/sweep.txt
done; done
