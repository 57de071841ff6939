OUT=gpurun_out/ab11; mkdir -p $OUT
for i in 1 2; do
TAG=passes python tools/time_sizes.py 65536 262144 16777216 >> $OUT/t.jsonl 2>&1
FFTC_LARGE=gpass TAG=gpass python tools/time_sizes.py 65536 262144 16777216 >> $OUT/t.jsonl 2>&1
done
