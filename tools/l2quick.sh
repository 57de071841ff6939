cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_direct_tc.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "graph or concurrent or direct or small_batches or config1 or multipass or candidate" 2>&1 | tail -3
