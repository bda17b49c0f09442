cd $GRAFT_REPO_ROOT
timeout 300 python tools/determinism_check.py 300
timeout 300 python tools/determinism_check.py 1024
timeout 900 python -m pytest tests/test_fuselage_gpu.py -q -m gpu --timeout 900 -s -k build_local 2>&1 | grep -v "^$" | tail -25 | cut -c1-600
timeout 900 python tools/bench_variance.py
