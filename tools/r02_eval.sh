# Round-2 evaluation pass on one B200: tests, smoke, bench lines (headline with c3/c4 sub-records,
# C1, reference arm), the ncu launch list of the bench command, per-job ncu lists, full captures.
OUT=gpurun_out/${TAG:-r02}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider 2>&1 | tail -15 > $OUT/pytest_gpu.txt
fi
python __graft_entry__.py --smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --workload c1 --no-cpu --no-e2e > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err
timeout 900 python bench.py --workload c5 --c5-loopback 8 --steps 5 --no-cpu --no-e2e > $OUT/bench_c5_lb8.json 2> $OUT/bench_c5.err
# launch list of the bench command (kernel time + DRAM bytes per launch)
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 900 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench.csv $CMD > $OUT/ncu_bench.log 2>&1
for w in c2 c3 c4; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/jobs_$w.csv python tools/ncu_jobs.py run --workload $w --map $OUT/jobs_${w}_map.json > $OUT/ncu_jobs_$w.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 2 -o $OUT/prof_n4096 python tools/prof_one.py 4096 > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass -c 2 -o $OUT/prof_pass python tools/prof_one.py 16777216 > $OUT/ncu_full2.log 2>&1
ls -la $OUT
