OUT=gpurun_out/ab13; mkdir -p $OUT
for i in 1 2; do
for g in 1 2 3 4 6 8; do
FFTC_PASS_GROUP=$g FFTC_PASS_GROUP_LONG=$g TAG=g$g python tools/time_sizes.py 65536 1048576 16777216 >> $OUT/t.jsonl 2>&1
done; done
