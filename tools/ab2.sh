OUT=gpurun_out/ab2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_candidate or config2 or config3 or config1 or small or ragged" 2>&1 | tail -3 > $OUT/pytest.txt
python tools/ab_kernels.py 4096 n4096_r16x16x16_t128x1 n4096_r16x16x16_t128x1_p16 n4096_r16x16x16_t128x1_p16sh n4096_r16x16x16_t256x1_p16 n4096_r16x16x16_t128x1_p16m5 n4096_r16x16x16_t256x1 > $OUT/ab4096.jsonl 2>&1
python tools/ab_kernels.py 2048 n2048_r16x16x8_t128x1_pk n2048_r16x16x8_t128x1 n2048_r16x16x8_t128x1_p16 > $OUT/ab2048.jsonl 2>&1
python tools/ab_kernels.py 1024 n1024_r32x32_t32x4 n1024_r32x32_t32x4_p16 > $OUT/ab1024.jsonl 2>&1
python tools/ab_kernels.py 512 n512_r32x16_t16x8 n512_r32x16_t16x8_p16 > $OUT/ab512.jsonl 2>&1
python tools/ab_kernels.py 256 n256_r16x16_t16x8 n256_r16x16_t16x8_p16 > $OUT/ab256.jsonl 2>&1
python tools/ab_kernels.py 2187 > $OUT/ab2187.jsonl 2>&1
python tools/ab_kernels.py 3125 > $OUT/ab3125.jsonl 2>&1
python tools/ab_kernels.py 1000 > $OUT/ab1000.jsonl 2>&1
python bench.py --no-cpu --no-e2e --no-extras > $OUT/bench.json 2>&1
python bench.py --workload c1 --no-cpu --no-e2e > $OUT/bench_c1.json 2>&1
