# 2^30 single GPU: pass splits and tile groups (time per transform, ms)
OUT=gpurun_out/ab30; mkdir -p $OUT
for i in 1 2; do
TAG=default python tools/time_sizes.py 1073741824 >> $OUT/t.jsonl 2>&1
for L in 10,10,10 11,10,9 12,9,9 9,9,12 12,10,8 8,10,12; do
for G in 3 6; do
FFTC_PASS_LOGS=$L FFTC_PASS_GROUP_LONG=$G TAG=s${L}_g$G python tools/time_sizes.py 1073741824 >> $OUT/t.jsonl 2>&1
done; done; done
