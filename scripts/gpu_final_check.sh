# final check at the head: full GPU suite and smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 600 > gpurun_out/r02_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke exit $?"; cat gpurun_out/r02_smoke.log | tail -1
