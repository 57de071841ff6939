OUT=gpurun_out/pg3; mkdir -p $OUT
python tools/prof_one.py 6561 12288 > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fftc_jit_pass -c 4 -o $OUT/prof_gpass python tools/prof_one.py 6561 12288 > $OUT/ncu.log 2>&1
ls -la $OUT
