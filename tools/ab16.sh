OUT=gpurun_out/ab16; mkdir -p $OUT
timeout 900 python -m pytest tests/test_jit.py tests/test_gpu_parity.py -q -x -k "jit or random" 2>&1 | tail -3 > $OUT/pytest.txt
for i in 1 2; do
FFTC_LIB_PATH=paper_2207_06803_b200/libfftc_ref.so TAG=ref python tools/time_sizes.py 11 13 61 121 143 176 704 1088 1369 2310 3328 >> $OUT/jit.jsonl 2>&1
TAG=new python tools/time_sizes.py 11 13 61 121 143 176 704 1088 1369 2310 3328 >> $OUT/jit.jsonl 2>&1
done
