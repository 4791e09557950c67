# randomized parity campaigns for the round-2 pair kernels (two homes per thread, window masks)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( echo "== SFB_RANDOM_CELLS=300: random cell-linked density / force vs the oracle (k_pairs_c two homes per thread, k_force_c)"
  SFB_RANDOM_CELLS=300 timeout 2400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "random_cell" 2>&1 | tail -2
  echo "== SFB_RANDOM_MASKED=200: random window-mask density -> masked force (1-3 slabs, reach 1/2, spread h, clumps) vs the oracle"
  SFB_RANDOM_MASKED=200 timeout 2400 python -m pytest tests/test_gpu_sharded.py -q -p no:cacheprovider -k "random_masked" 2>&1 | tail -2
) > gpurun_out/r02_random_cells.txt 2>&1
cat gpurun_out/r02_random_cells.txt
