# quick GPU iteration: parity (subset) + perf sweep (+ optional ncu of a workload)
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "small_batches or config1 or fourstep or special or n1" 2>&1 | tail -5
timeout 300 python tools/perf_sweep.py 2>&1 | tail -25
if [ -n "$NCU_WL" ]; then
python bench.py --workload $NCU_WL --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_$NCU_WL.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv --log-file gpurun_out/launches_$NCU_WL.csv python bench.py --workload $NCU_WL --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$NCU_WL.log 2>&1
fi
