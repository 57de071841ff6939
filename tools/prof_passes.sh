OUT=gpurun_out/pp; mkdir -p $OUT
python tools/prof_one.py 4194304 1048576 > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass -c 4 -o $OUT/prof_p22_p20 python tools/prof_one.py 4194304 1048576 > $OUT/ncu1.log 2>&1
export FFTC_PASS_LOGS=12,12 FFTC_PASS_FIRST=p4096_r16x16x16_c2b3 FFTC_PASS=p4096_r16x16x16_c4b1
python tools/prof_one.py 16777216 > $OUT/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass -c 2 -o $OUT/prof_p24_4096x2 python tools/prof_one.py 16777216 > $OUT/ncu2.log 2>&1
ls -la $OUT
