OUT=gpurun_out/ab21; mkdir -p $OUT
S="60 105 210 1000 2187 3125 64 256 512 1024 2048 4096"
for i in 1 2; do
TAG=compiled python tools/time_sizes.py $S >> $OUT/t.jsonl 2>&1
FFTC_FORCE_JIT=1 TAG=jit python tools/time_sizes.py $S >> $OUT/t.jsonl 2>&1
done
