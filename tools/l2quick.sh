cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_direct_tc.py -v -m gpu -p no:cacheprovider --timeout 60 -x > gpurun_out/direct.log 2>&1
grep -E "^E|FAILED|passed|failed" gpurun_out/direct.log | head -20
python - <<'PY'
import sys, torch; sys.path.insert(0,'.')
import paper_2207_06803_b200 as fftc
for N in (16, 32):
    b=(1<<26)//N
    x=torch.randn(N*b,dtype=torch.complex64,device='cuda'); y=torch.empty_like(x)
    for mk in (lambda: fftc.Plan.direct(N,b,-1), lambda: fftc.Plan(N,b,-1)):
        p=mk()
        for _ in range(3): p.execute(x,y)
        ts=[]
        for _ in range(10):
            a=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
            a.record(); p.execute(x,y); e.record(); e.synchronize(); ts.append(a.elapsed_time(e))
        ts.sort(); t=ts[5]
        print(N, b, 'us', round(t*1e3,1), 'GB/s', round(16*N*b/t/1e6,1), p.describe()[:90])
        p.close()
PY
