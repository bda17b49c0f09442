cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gmres_gpu.py -q -m gpu --timeout 900 -x 2>&1 | tail -15
