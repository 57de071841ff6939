OUT=gpurun_out/ab18; mkdir -p $OUT
S="12 24 48 96 120 192 360 500 729 1344 2401 3000 4000 1536 3072 640 768 2000"
for i in 1 2; do
TAG=generic python tools/time_sizes.py $S >> $OUT/t.jsonl 2>&1
FFTC_SMOOTH_JIT=1 TAG=jit python tools/time_sizes.py $S >> $OUT/t.jsonl 2>&1
done
FFTC_SMOOTH_JIT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "generic or all_smooth" 2>&1 | tail -3 > $OUT/pytest.txt
