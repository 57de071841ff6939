cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "l2 or multipass or fourstep_small or execute_host or describe or config4" 2>&1 | tail -3
for n in 13 14 15 16 17 18 19 20 21 22 23 24; do for m in passes fourstep; do FFTC_LARGE=$m timeout 100 python tools/l2sweep.py one $n $(( (1<<28) >> n )) | cut -c1-120; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass -c 2 -o gpurun_out/prof_pass16 python tools/l2sweep.py one 16 1024 > gpurun_out/ncu_p.log 2>&1
tail -1 gpurun_out/ncu_p.log
