# compute-sanitizer over the round-2 pair kernels (two-homes density, window masks, masked force) and the shard
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SAN="compute-sanitizer --error-exitcode 9"
( for tool in memcheck racecheck synccheck; do
    echo "== $tool: cell density / force (two homes per thread, reach 1-4, spread h, ghosts), window masks (1-3 slabs, clumps, ghosts), single-rank shard"
    timeout 1500 $SAN --tool $tool python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_sharded.py -k "cells_vs_oracle or reach_3 or homes_and or coincident or masked or single_rank or uniform" 2>&1 | tail -3
    echo "exit $?"
  done ) > gpurun_out/r02_sanitizer_pairs.txt 2>&1
cat gpurun_out/r02_sanitizer_pairs.txt
