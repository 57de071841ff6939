cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_direct_tc.py -q -m gpu -p no:cacheprovider --timeout 60 -x 2>&1 | tail -1
for g in 296; do FFTC_DIRECT_GRID=$g python - <<'PY'
import sys, os, torch; sys.path.insert(0,'.')
import paper_2207_06803_b200 as fftc
x=torch.randn(1<<26,dtype=torch.complex64,device='cuda'); y=torch.empty_like(x)
for N in (16,32):
    b=(1<<26)//N; p=fftc.Plan.direct(N,b,-1)
    for _ in range(3): p.execute(x,y)
    ts=[]
    for _ in range(10):
        a=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        a.record(); p.execute(x,y); e.record(); e.synchronize(); ts.append(a.elapsed_time(e))
    ts.sort(); t=ts[5]; print(os.environ['FFTC_DIRECT_GRID'], N, round(t*1e3,1), 'us', round(16*N*b/t/1e6), 'GB/s')
    p.close()
PY
done
