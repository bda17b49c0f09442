cd $GRAFT_REPO_ROOT
for i in 1 2; do
python bench.py --steps 5 --warmup 3 --no-cpu --no-offline --no-per-order --no-parity > gpurun_out/fresh$i.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/fresh$i.json').read().strip().splitlines()[-1]); print('run $i', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
done
