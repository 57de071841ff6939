cd $GRAFT_REPO_ROOT
for k in p256_r16x16_b2m2 p256_r16x16_b2m1; do for n in 16 24; do FFTC_PASS=$k timeout 100 python tools/l2sweep.py one $n $(( (1<<28) >> n )) | cut -c1-110; done; done
for k in p128_r16x8 p128_r16x8_b2m2; do for n in 14 21; do FFTC_PASS=$k timeout 100 python tools/l2sweep.py one $n $(( (1<<28) >> n )) | cut -c1-110; done; done
for k in p512_r16x32_c8t32 p512_r32x16_c8m2 p512_r16x32_c8t32m1; do FFTC_PASS=$k timeout 100 python tools/l2sweep.py one 18 1024 | cut -c1-110; done
for k in p64_r8x8 p64_r8x8_m4; do FFTC_PASS=$k timeout 100 python tools/l2sweep.py one 13 32768 | cut -c1-110; done
