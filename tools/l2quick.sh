cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_graph.py -k l2 -v -m gpu -p no:cacheprovider --timeout 120 2>&1 | grep -E "PASS|FAIL|^E " | head -30
