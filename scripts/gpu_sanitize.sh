# compute-sanitizer over the edge-case parity tests (1 GPU): memcheck (ragged tails, shifted / wide
# records, random schemas, binning), racecheck and synccheck (staged shared-memory kernels).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "ragged or shifted or wide or random_schemas or zero_records or sequence_ragged or bin_particles" -p no:cacheprovider > gpurun_out/sanitize.log 2>&1
echo "memcheck $?"
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "sequence_ragged or random_schemas_match_oracle[0] or random_schemas_match_oracle[1] or zero_records" -p no:cacheprovider > gpurun_out/race.log 2>&1
echo "racecheck $?"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "sequence_ragged or random_schemas_match_oracle[2]" -p no:cacheprovider > gpurun_out/sync.log 2>&1
echo "synccheck $?"
timeout 2200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q \
  -k "(cells or density or force or uniform) and not across_processes and not peer" -p no:cacheprovider > gpurun_out/sanitize2.log 2>&1
echo "memcheck cells $?"
