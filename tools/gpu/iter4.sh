cd $GRAFT_REPO_ROOT
timeout 600 python tools/prof_orth.py --grouped | cut -c1-300
timeout 1200 python -m pytest tests/test_fuselage_gpu.py tests/test_linalg_gpu.py tests/test_fdm_gpu.py tests/test_dist_gpu.py -q -m gpu --timeout 900 -s 2>&1 | grep -v "^\.\|^$" | tail -12
