# Time pass-kernel combinations (first pass x later passes) per size; dev tool.
# bash tools/pass_matrix.sh > gpurun_out/pass_matrix.jsonl
run() { FFTC_PASS_FIRST=$1 FFTC_PASS=$2 TAG="$1|$2" python tools/time_sizes.py $3; }
for r in 1 2; do
for f in p256_r16x16_b2m2 p256_r16x16_b3m2; do for l in p256_r16x16_b2m2 p256_r16x16_b3m2; do run $f $l "65536 16777216"; done; done
for f in p1024_r32x32_c8b1m2 p1024_r32x32_c8b2 p1024_r32x32_c8b3; do for l in p1024_r32x32_c8b1m2 p1024_r32x32_c8b2 p1024_r32x32_c8b3; do run $f $l 1048576; done; done
for f in p1024_r32x32_c8b2 p1024_r32x32_c8b3; do for l in p1024_r32x32_c8b2,p256_r16x16_b2m2 p1024_r32x32_c8b3,p256_r16x16_b2m2 p1024_r32x32_c8b3,p256_r16x16_b3m2 p1024_r32x32_c8b2,p256_r16x16_b3m2; do run $f $l "268435456 33554432"; done; done
for f in p512_r16x32_c8t32 p512_r16x32_c8t32b3; do for l in p512_r16x32_c8t32 p512_r16x32_c8t32b3; do run $f $l 262144; done; done
for f in p128_r16x8 p128_r16x8_b4m3; do for l in p256_r16x16_b2m2 p256_r16x16_b3m2; do run $f $l "32768 8192"; done; done
done
