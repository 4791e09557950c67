# randomized parity campaigns at the round-2 head (conversion schemas, in-place kick/drift layouts, buffer-mode
# density/force, fused gather+kernel compositions; the live reference or the oracle as the checker)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # run <env> <count> <-k expr> <label>
  echo "== $1=$2: $4"
  env $1=$2 timeout 2400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$3" 2>&1 | tail -1
}
( run SFB_RANDOM_SCHEMAS 3000 "random_schemas_match" "random conversion schemas vs the oracle"
  run SFB_RANDOM_KD 2000 "random_kick_drift_layouts" "random in-place kick/drift layouts vs the live reference"
  run SFB_RANDOM_DF 600 "random_density_force_layouts" "random buffer-mode density/force layouts vs the live reference"
  run SFB_RANDOM_FUSED 2000 "random_fused_gather" "random fused gather+kernel compositions vs the live reference"
) > gpurun_out/r02_random_campaign.txt 2>&1
cat gpurun_out/r02_random_campaign.txt
