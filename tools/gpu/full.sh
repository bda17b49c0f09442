cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --durations=15 > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_full.log
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_full.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')})
print('roofline', d['roofline']['frac'], 'e2e', d['e2e']['value'], 'parity', d['parity'])
for k,v in (d['per_order'] or {}).items(): print(k, {kk: vv for kk, vv in v.items() if kk != 'parity'}, (v.get('parity') or {}).get('max_tf_rel_err'))
print('cpu', d['cpu_baseline']['value'], d['cpu_baseline']['cores'])
o=d['offline']; print({k:v for k,v in o.items() if 'pipeline' in k or 'fuselage' in k})
PY
