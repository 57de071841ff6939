OUT=gpurun_out/ab15; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_candidate and (4096 or 2048 or 2187 or 3125 or 1000)" 2>&1 | tail -3 > $OUT/pytest.txt
python tools/ab_kernels.py 4096 n4096_r16x16x16_t128x1 n4096_r16x16x16_t128x1_na > $OUT/na.jsonl 2>&1
python tools/ab_kernels.py 2187 n2187_r27x9x9_t128x1 n2187_r27x9x9_t128x1_na >> $OUT/na.jsonl 2>&1
python tools/ab_kernels.py 3125 n3125_r25x5x25_t128x1_pk n3125_r25x5x25_t128x1_pk_na n3125_r25x5x25_t128x1_na >> $OUT/na.jsonl 2>&1
python tools/ab_kernels.py 1000 n1000_r10x10x10_t100x2_pk n1000_r10x10x10_t100x2_pk_na >> $OUT/na.jsonl 2>&1
python tools/ab_kernels.py 2048 n2048_r16x16x8_t128x1_pk n2048_r16x16x8_t128x1_pk_na >> $OUT/na.jsonl 2>&1
