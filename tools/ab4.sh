OUT=gpurun_out/ab4; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_jit.py tests/test_expr.py -q -x 2>&1 | tail -3 > $OUT/pytest.txt
for i in 1 2 3; do
  FFTC_LIB_PATH=paper_2207_06803_b200/libfftc_ref.so TAG=ref python tools/time_sizes.py 60 105 210 2187 6561 19683 >> $OUT/dft3.jsonl 2>&1
  TAG=new python tools/time_sizes.py 60 105 210 2187 6561 19683 >> $OUT/dft3.jsonl 2>&1
done
