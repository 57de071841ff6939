OUT=gpurun_out/ab12; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gpass" 2>&1 | tail -3 > $OUT/pytest.txt
python - > $OUT/par.txt 2>&1 <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth, paper_2207_06803_b200 as fftc
os.environ['FFTC_LARGE'] = 'gpass'
for N, lens in [(1 << 24, '4096,4096'), (1 << 22, '4096,1024'), (1 << 21, '2048,1024')]:
    os.environ['FFTC_GPASS_LENGTHS'] = lens
    x = synth.uniform_c64(N, 2, seed=3)
    for sign in (-1, 1):
        with fftc.Plan(N, 2, sign) as p:
            y = p(torch.from_numpy(x).cuda()).cpu().numpy()
            d = p.describe()
        ref = np.fft.fft(x.astype(np.complex128), axis=1) if sign < 0 else np.fft.ifft(x.astype(np.complex128), axis=1) * N
        err = np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1)
        print(N, lens, sign, err.max(), oracle.tolerance(N), d[:100])
PY
for i in 1 2; do
TAG=passes python tools/time_sizes.py 2097152 4194304 8388608 16777216 >> $OUT/t.jsonl 2>&1
FFTC_LARGE=gpass FFTC_GPASS_LENGTHS=2048,1024 TAG=g2048x1024 python tools/time_sizes.py 2097152 >> $OUT/t.jsonl 2>&1
FFTC_LARGE=gpass FFTC_GPASS_LENGTHS=4096,1024 TAG=g4096x1024 python tools/time_sizes.py 4194304 >> $OUT/t.jsonl 2>&1
FFTC_LARGE=gpass FFTC_GPASS_LENGTHS=2048,2048 TAG=g2048x2048 python tools/time_sizes.py 4194304 >> $OUT/t.jsonl 2>&1
FFTC_LARGE=gpass FFTC_GPASS_LENGTHS=4096,2048 TAG=g4096x2048 python tools/time_sizes.py 8388608 >> $OUT/t.jsonl 2>&1
FFTC_LARGE=gpass FFTC_GPASS_LENGTHS=4096,4096 TAG=g4096x4096 python tools/time_sizes.py 16777216 >> $OUT/t.jsonl 2>&1
done
