cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_lu_gpu.py -q -m gpu --timeout 300 2>&1 | tail -4
timeout 600 python tools/bench_lu.py 4641 8102
