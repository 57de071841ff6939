OUT=gpurun_out/ab25; mkdir -p $OUT
python tools/ab_kernels.py 60 n60_r4x15_t4x16d n60_r4x15_t4x16 n60_r4x15_t4x32 --rounds 8 >> $OUT/ab.jsonl 2>&1
python tools/ab_kernels.py 4096 n4096_r16x16x16_t128x1_na n4096_r16x16x16_t256x1 n4096_r16x16x16_t256x1_na n4096_r16x16x16_t256x1_pk --rounds 8 >> $OUT/ab.jsonl 2>&1
python tools/ab_kernels.py 1024 n1024_r32x32_t32x4 n1024_r32x32_t32x2 n1024_r32x32_t32x4_shfl --rounds 8 >> $OUT/ab.jsonl 2>&1
python tools/ab_kernels.py 256 n256_r16x16_t16x8 n256_r16x16_t16x16 n256_r16x16_t16x8_shfl --rounds 8 >> $OUT/ab.jsonl 2>&1
python tools/ab_kernels.py 512 n512_r32x16_t16x8 n512_r32x16_t16x4 --rounds 8 >> $OUT/ab.jsonl 2>&1
