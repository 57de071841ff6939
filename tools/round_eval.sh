# Full evaluation pass on one B200: tests, smoke, bench lines, ncu launch lists and full captures.
OUT=gpurun_out/${TAG:-eval}
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider 2>&1 | tail -5 > $OUT/pytest_gpu.txt
python __graft_entry__.py --smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
python bench.py --impl reference > $OUT/ref_c2.json 2> $OUT/ref_c2.err
for w in c1 c3 c4 c5; do python bench.py --workload $w --no-e2e --no-cpu > $OUT/bench_$w.json 2> $OUT/bench_$w.err; done
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_c2.log 2>&1
python bench.py --workload c4 --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 100 --csv --log-file $OUT/launches_c4.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_c4.log 2>&1
python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 100 --csv --log-file $OUT/launches_c3.csv python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:\\(int\\)4096" -c 1 -o $OUT/prof_n4096 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass -c 2 -o $OUT/prof_pass python bench.py --workload c4 --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/ncu_full4.log 2>&1
ls -la $OUT
