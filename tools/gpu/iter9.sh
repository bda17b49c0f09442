cd $GRAFT_REPO_ROOT
timeout 600 python tools/prof_orth_kernels.py 2>&1 | grep -v Warn | head -12 | cut -c1-200
timeout 900 python -m pytest tests/test_linalg_gpu.py tests/test_dist_gpu.py tests/test_fdm_gpu.py -q -m gpu --timeout 900 2>&1 | tail -3
