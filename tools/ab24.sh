OUT=gpurun_out/ab24; mkdir -p $OUT
for N in 8 16 32 64 128 256 512 1024 2048 4096 60 105 210 1000 2187 3125; do
  python tools/ab_kernels.py $N --rounds 4 --reps 12 >> $OUT/all.jsonl 2>&1
done
