cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "multipass or l2 or fourstep_small or pass_candidate or config4" 2>&1 | tail -1
python bench.py --workload c4 --no-e2e --no-cpu --steps 10 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])
for j in d['per_job']: print(j['N'], j['sign'], j['us'], j['eff_GBs'])"
