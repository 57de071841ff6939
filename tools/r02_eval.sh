# Round-2 evaluation pass on one B200: tests, smoke, bench (default line with c3/c4 sub-records),
# per-job ncu launch lists for c2/c3/c4.
OUT=gpurun_out/${TAG:-r02}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider 2>&1 | tail -15 > $OUT/pytest_gpu.txt
fi
python __graft_entry__.py --smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --gpus 1 --workload c1 --no-cpu --no-e2e > $OUT/bench_c1.json 2> $OUT/bench_c1.err
for w in c2 c3 c4; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/jobs_$w.csv python tools/ncu_jobs.py run --workload $w --map $OUT/jobs_${w}_map.json > $OUT/ncu_jobs_$w.log 2>&1
done
ls -la $OUT
