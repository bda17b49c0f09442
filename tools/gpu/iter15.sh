cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fdm_gpu.py tests/test_dist_gpu.py tests/test_determinism_gpu.py tests/test_gmres_gpu.py tests/test_lu_gpu.py -q -m gpu --timeout 900 2>&1 | tail -3
timeout 600 python tools/prof_orth.py | cut -c1-200
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-per-order --no-parity > gpurun_out/bench_off.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_off.json').read().strip().splitlines()[-1]); o=d['offline']; print({k:v for k,v in o.items() if 'pipeline' in k or k.startswith('fuselage_b') or k.startswith('fuselage_s')})"
