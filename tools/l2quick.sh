cd $GRAFT_REPO_ROOT
for cfg in "32 3" "8 3" "16 4" "64 3" "128 2" "16 3"; do set -- $cfg; FFTC_HOST_CHUNK_MB=$1 FFTC_HOST_DEPTH=$2 python - <<'PY'
import sys, os, time, torch; sys.path.insert(0,'.')
import paper_2207_06803_b200 as fftc
N=1024; b=(1<<26)//N
x=torch.randn(N*b,dtype=torch.complex64).pin_memory(); y=torch.empty_like(x).pin_memory()
p=fftc.Plan(N,b,-1); p.execute_host(x,y)
t=time.perf_counter()
for _ in range(5): p.execute_host(x,y)
t=(time.perf_counter()-t)/5
print(os.environ['FFTC_HOST_CHUNK_MB'], os.environ['FFTC_HOST_DEPTH'], 'ms', round(t*1e3,2), 'GB/s per direction', round(8*N*b/t/1e9,1))
PY
done
