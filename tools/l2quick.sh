cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist.py -v -m gpu -p no:cacheprovider --timeout 300 -x > gpurun_out/dist.log 2>&1
grep -E "^E|FAILED|passed|failed" gpurun_out/dist.log | head -20
