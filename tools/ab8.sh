OUT=gpurun_out/ab8; mkdir -p $OUT
for i in 1 2; do
for c in none 100 86 72 58 44; do
  if [ $c = none ]; then TAG=carve_$c python tools/time_sizes.py 4096 2048 2187 3125 1000 >> $OUT/carve.jsonl 2>&1;
  else FFTC_CARVEOUT=$c TAG=carve_$c python tools/time_sizes.py 4096 2048 2187 3125 1000 >> $OUT/carve.jsonl 2>&1; fi
done; done
