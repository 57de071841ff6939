# cluster 4096-long pass candidates: parity against numpy (fp64) and timing against the default plans
OUT=gpurun_out/ab26; mkdir -p $OUT
for PASSN in cp4096_q4_r32x32_c8b2; do
FFTC_PASS=$PASSN python - >> $OUT/par.txt 2>&1 <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth, paper_2207_06803_b200 as fftc
for N, logs, batch in [(1 << 24, '12,12', 2), (1 << 22, '12,10', 3), (1 << 20, '12,8', 5)]:
    os.environ['FFTC_PASS_LOGS'] = logs
    x = synth.uniform_c64(N, batch, seed=3)
    for sign in (-1, 1):
        with fftc.Plan(N, batch, sign) as p:
            y = p(torch.from_numpy(x).cuda()).cpu().numpy()
            d = p.describe()
        ref = np.fft.fft(x.astype(np.complex128), axis=1) if sign < 0 else np.fft.ifft(x.astype(np.complex128), axis=1) * N
        err = np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1)
        print(N, logs, sign, err.max(), oracle.tolerance(N), d[:120], flush=True)
PY
done
for i in 1 2; do
TAG=default python tools/time_sizes.py 16777216 4194304 >> $OUT/t.jsonl 2>&1
for PASSN in cp4096_q4_r32x32_c8b2; do
FFTC_PASS=$PASSN FFTC_PASS_LOGS=12,12 TAG=$PASSN python tools/time_sizes.py 16777216 >> $OUT/t.jsonl 2>&1
FFTC_PASS=$PASSN FFTC_PASS_LOGS=12,10 TAG=$PASSN python tools/time_sizes.py 4194304 >> $OUT/t.jsonl 2>&1
done
done
