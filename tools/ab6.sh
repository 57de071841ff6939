OUT=gpurun_out/ab6; mkdir -p $OUT
FFTC_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --no-cpu --no-extras > $OUT/bench_g2.json 2> $OUT/bench_g2.err
FFTC_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 4 --steps 5 --no-cpu --no-extras --no-e2e > $OUT/bench_g4.json 2> $OUT/bench_g4.err
FFTC_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --workload c3 --no-cpu --no-e2e > $OUT/bench_g2c3.json 2> $OUT/bench_g2c3.err
