OUT=gpurun_out/ab9; mkdir -p $OUT
for i in 1 2 3; do
FFTC_LIB_PATH=paper_2207_06803_b200/libfftc_ref.so TAG=ref python tools/time_sizes.py 60 105 210 2187 >> $OUT/dft3.jsonl 2>&1
TAG=new python tools/time_sizes.py 60 105 210 2187 >> $OUT/dft3.jsonl 2>&1
done
