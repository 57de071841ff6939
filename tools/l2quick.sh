cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "multipass or l2 or fourstep_small or pass_candidate or config4 or describe" 2>&1 | tail -1
for i in 1 2; do for n in 16 20 24; do timeout 100 python tools/l2sweep.py one $n $(( (1<<28) >> n )) | cut -c1-60; done; done
