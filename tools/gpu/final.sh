cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --durations=10 > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"
tail -14 gpurun_out/pytest_full.log
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','gpu_launches')})
print('roofline', d['roofline']['frac'], 'e2e', d['e2e']['value'], 'parity', d['parity']['max_tf_rel_err'], d['parity']['max_dspl_db'])
for k,v in (d['per_order'] or {}).items(): print(k, v.get('value'), v.get('frac'), (v.get('parity') or {}).get('max_tf_rel_err'))
print('cpu', d['cpu_baseline']['value'], d['cpu_baseline']['cores'])
o=d['offline']; print({k:v for k,v in o.items() if ('pipeline' in k and 'first' not in k) or k in ('fuselage_sweep_s','fuselage_build_s','fuselage_build_same_points')})
r=json.loads(open('gpurun_out/bench_ref.json').read().strip().splitlines()[-1]); print('ref', r['value'], r['config'] == d['config'])
PY
