OUT=gpurun_out/ab10; mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider 2>&1 | tail -15 > $OUT/pytest_gpu.txt
python __graft_entry__.py --smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --workload c1 --no-cpu --no-e2e > $OUT/bench_c1.json 2> $OUT/bench_c1.err
python tools/prof_one.py 6561 > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fftc_jit_pass -c 2 -o $OUT/prof_gpass python tools/prof_one.py 6561 > $OUT/ncu.log 2>&1
