cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_jit.py tests/test_gpu_parity.py -v -m gpu -p no:cacheprovider --timeout 120 -k "jit or boundary" > gpurun_out/jit_gpu.log 2>&1
grep -E "^E|FAILED|passed|failed" gpurun_out/jit_gpu.log | tail -15
python - <<'PY'
import sys, torch; sys.path.insert(0,'.')
import paper_2207_06803_b200 as fftc
for N in (11, 13, 61, 143, 3328):
    b=(1<<26)//N
    x=torch.randn(N*b,dtype=torch.complex64,device='cuda'); y=torch.empty_like(x)
    p=fftc.Plan(N,b,-1)
    for _ in range(3): p.execute(x,y)
    ts=[]
    for _ in range(5):
        a=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        a.record(); p.execute(x,y); e.record(); e.synchronize(); ts.append(a.elapsed_time(e))
    ts.sort(); t=ts[2]
    print(N, b, 'us', round(t*1e3,1), 'GB/s', round(16*N*b/t/1e6,1), p.describe())
PY
