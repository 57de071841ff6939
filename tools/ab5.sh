OUT=gpurun_out/ab5; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_jit.py tests/test_expr.py tests/test_gpu_graph.py -q -x -k "gpass or jit or expr or graph or random_large" 2>&1 | tail -5 > $OUT/pytest.txt
python tools/time_sizes.py 6561 19683 100000 1000000 12288 61440 45056 59049 > $OUT/times.jsonl 2>&1
