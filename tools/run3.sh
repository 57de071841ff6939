set -x
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_c2.json 2>&1; echo ref rc=$?
python bench.py --workload c3 --no-e2e --no-cpu > gpurun_out/bench_c3.json 2>&1
python bench.py --workload c4 --no-e2e --no-cpu > gpurun_out/bench_c4.json 2>&1
python bench.py --workload c1 --no-e2e --no-cpu > gpurun_out/bench_c1.json 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused_batch -s 18 -c 1 -o gpurun_out/prof_n4096 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused_batch -s 8 -c 1 -o gpurun_out/prof_n128 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
