# GPU suite + quick bench A/B (L2 persistence on/off) + ROM accuracy survey
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --durations=30 > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?"
tail -45 gpurun_out/pytest_r2b.log
for p in 0 1; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-offline --no-cpu --no-per-order --l2-persist $p > gpurun_out/bench_l2_$p.json 2>&1; echo "bench l2=$p rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_l2_$p.json').read().strip().splitlines()[-1]); print('l2',$p,d['value'],d['roofline']['frac'],d['e2e']['value'])"
done
timeout 900 python tools/rom_accuracy.py > gpurun_out/rom_accuracy.json 2>&1; echo "rom acc rc=$?"
cat gpurun_out/rom_accuracy.json | tail -5
