cd $GRAFT_REPO_ROOT
cat > /tmp/g.py <<'PY'
import sys, torch; sys.path.insert(0,'.')
import paper_2207_06803_b200 as fftc
N=59049; b=1136
x=torch.randn(N*b,dtype=torch.complex64,device='cuda'); y=torch.empty_like(x)
p=fftc.Plan(N,b,-1)
for _ in range(2): p.execute(x,y)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gpass -s 2 -c 2 -o gpurun_out/prof_gpass python /tmp/g.py > gpurun_out/ncu_g.log 2>&1
tail -2 gpurun_out/ncu_g.log
