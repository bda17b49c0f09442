cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fuselage_gpu.py tests/test_dist_gpu.py -q -m gpu --timeout 900 -s 2>&1 | grep "GPU build\|passed\|failed\|Error" | cut -c1-400
timeout 600 python tools/prof_orth_kernels.py 2>&1 | head -40
for i in 1 2; do timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-offline --no-per-order > gpurun_out/bench_rep$i.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/bench_rep$i.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['parity']['max_tf_rel_err'])"; done
