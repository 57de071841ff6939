OUT=gpurun_out/ab3; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_candidate and (64 or 256 or 1024)" 2>&1 | tail -3 > $OUT/pytest.txt
python tools/ab_kernels.py 64 n64_r8x8_t8x8d n64_r8x8_t8x8_shfl n64_r8x8_t8x16_shfl > $OUT/shfl64.jsonl 2>&1
python tools/ab_kernels.py 256 n256_r16x16_t16x8 n256_r16x16_t16x8_shfl n256_r16x16_t16x16_shfl > $OUT/shfl256.jsonl 2>&1
python tools/ab_kernels.py 1024 n1024_r32x32_t32x4 n1024_r32x32_t32x4_shfl > $OUT/shfl1024.jsonl 2>&1
python bench.py --workload c4 --no-cpu --no-e2e --steps 10 > $OUT/bench_c4.json 2>&1
for s in "" "10,10,10" "12,9,9" "11,10,9"; do TAG="logs=$s" FFTC_PASS_LOGS=$s python tools/time_sizes.py 1073741824 >> $OUT/c5_splits.jsonl 2>&1; done
