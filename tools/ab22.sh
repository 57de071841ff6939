OUT=gpurun_out/ab22; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_jit.py tests/test_gpu_parity.py tests/test_expr.py -q -x -k "jit or gpass or random or 7smooth or expr or small_batches" 2>&1 | tail -3 > $OUT/pytest.txt
S="48 192 768 1536 3072 640 2000 4000 2401 143 1088 1369 2310 3328"
for i in 1 2; do
FFTC_LIB_PATH=paper_2207_06803_b200/libfftc_ref.so TAG=ref python tools/time_sizes.py $S 6561 12288 100000 45056 >> $OUT/t.jsonl 2>&1
TAG=new python tools/time_sizes.py $S 6561 12288 100000 45056 >> $OUT/t.jsonl 2>&1
done
