cd $GRAFT_REPO_ROOT
CHUNKS=4,8,16,32 GRIDS=0,148,296 timeout 900 python tools/l2sweep.py 2>&1 | tail -30
FFTC_L2_CHUNK_MB=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_l2 -c 1 -o gpurun_out/prof_l2_16 python tools/l2sweep.py one 16 1024 > gpurun_out/ncu_l2.log 2>&1
tail -3 gpurun_out/ncu_l2.log
