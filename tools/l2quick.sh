cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider --timeout 300 -x -k "multipass or describe" 2>&1 | tail -1
for n in 25 26 27 28; do timeout 100 python tools/l2sweep.py one $n $(( (1<<28) >> n )) | cut -c1-70; done
