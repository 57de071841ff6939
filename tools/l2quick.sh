cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py --workload c4 --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c4.json; head -c 300 gpurun_out/bench_c4.json; echo
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c4.json').read())
for j in d['per_job']: print(j)
PY
