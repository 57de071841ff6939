OUT=gpurun_out/ab1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_candidate and (4096 or 2048 or 2187 or 3125 or 1000)" 2>&1 | tail -3 > $OUT/pytest.txt
python tools/ab_kernels.py 4096 n4096_r16x16x16_t128x1 n4096_r16x16x16_t128x1_sh n4096_r16x16x16_t128x1_v n4096_r16x16x16_t128x1_vsh n4096_r16x16x16_t128x1_vshl n4096_r16x16x16_t128x1_l n4096_r16x16x16_t128x1_pk_vsh n4096_r16x16x16_t256x1 > $OUT/ab4096.jsonl 2>&1
python tools/ab_kernels.py 2048 n2048_r16x16x8_t128x1_pk n2048_r16x16x8_t128x1 n2048_r16x16x8_t128x1_vsh > $OUT/ab2048.jsonl 2>&1
python tools/ab_kernels.py 2187 n2187_r27x9x9_t128x1 n2187_r27x9x9_t81x2 n2187_r27x9x9_t81x2_sh n2187_r27x9x9_t81x2_shl n2187_r27x9x9_t128x1_l n2187_r27x9x9_t81x2_pk_sh > $OUT/ab2187.jsonl 2>&1
python tools/ab_kernels.py 3125 n3125_r25x5x25_t128x1_pk n3125_r25x5x25_t125x2 n3125_r25x5x25_t125x2_sh n3125_r25x5x25_t125x2_pk_sh > $OUT/ab3125.jsonl 2>&1
python tools/ab_kernels.py 1000 n1000_r10x10x10_t100x2_pk n1000_r10x10x10_t50x2 n1000_r10x10x10_t50x2_vsh n1000_r10x10x10_t100x2_v n1000_r10x10x10_t50x2_pk_vsh n1000_r10x10x10_t100x2_pk_v > $OUT/ab1000.jsonl 2>&1
python bench.py --workload c1 --no-cpu --no-e2e > $OUT/bench_c1.json 2>&1
