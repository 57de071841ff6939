cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "candidate" 2>&1 | tail -1
python tools/tune.py 4096 2048
