cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_expr.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "gpass or gpu_expr" 2>&1 | tail -1
timeout 900 python tools/bench_extra.py 2>&1 | grep gpass | cut -c1-120
