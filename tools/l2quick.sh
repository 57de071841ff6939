cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -v -m gpu -p no:cacheprovider --timeout 120 > gpurun_out/gpu_all.log 2>&1
grep -E "^E|FAILED|passed|failed" gpurun_out/gpu_all.log | tail -15
