cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_jit.py tests/test_gpu_parity.py tests/test_expr.py -q -m gpu -p no:cacheprovider --timeout 300 -k "jit or gpass or gpu_expr or boundary" 2>&1 | tail -15 | grep -E "^E|FAILED|passed|failed"
timeout 900 python tools/bench_extra.py 2>&1 | grep gpass | cut -c1-230
