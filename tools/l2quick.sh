cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gpass or describe" 2>&1 | tail -30 | grep -E "^E|passed|failed"
for N in 59049 100000 1000000; do python - <<PY
import sys, torch, math; sys.path.insert(0,'.')
import paper_2207_06803_b200 as fftc
N=$N; b=(1<<28)//N
x=torch.randn(N*b,dtype=torch.complex64,device='cuda'); y=torch.empty_like(x)
p=fftc.Plan(N,b,-1)
for _ in range(3): p.execute(x,y)
ts=[]
for _ in range(5):
    a=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    a.record(); p.execute(x,y); e.record(); e.synchronize(); ts.append(a.elapsed_time(e))
ts.sort(); t=ts[2]; L=p.launches()
print(N, b, 'ms', round(t,3), 'HBM GB/s per pass', round(16*N*b*L/t/1e6,1), p.describe())
PY
done
