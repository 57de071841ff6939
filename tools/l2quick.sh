cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -v -m gpu -p no:cacheprovider --timeout 300 -k "2p31" 2>&1 | grep -E "PASS|FAIL|^E" | head
