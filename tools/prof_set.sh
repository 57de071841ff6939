# ncu --set full of the second launch of each size's kernels.  SIZES env var.
python tools/prof_one.py $SIZES > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fused|k_colx|k_rows|k_pass" -o gpurun_out/prof_$TAG python tools/prof_one.py $SIZES > gpurun_out/prof_$TAG.log 2>&1
tail -3 gpurun_out/prof_$TAG.log
