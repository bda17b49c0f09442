cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_lu_gpu.py -q -m gpu --timeout 300 -x 2>&1 | tail -15
timeout 600 python tools/bench_lu.py
