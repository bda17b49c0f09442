cd $GRAFT_REPO_ROOT
timeout 600 python tools/prof_orth.py --grouped
timeout 1200 python -m pytest tests/test_fuselage_gpu.py -q -m gpu --timeout 900 -s 2>&1 | tail -8
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-per-order --no-parity > gpurun_out/bench_off.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_off.json').read().strip().splitlines()[-1]); o=d['offline']; print({k:v for k,v in o.items() if 'pipeline' in k or k.endswith('_r')})"
tail -3 gpurun_out/bench_off.json | cut -c1-2000
