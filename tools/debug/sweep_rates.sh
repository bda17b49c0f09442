# sweep throughput at several orders (device-resident, no e2e/cpu/offline legs)
for r in ${@:-256 400 1024 2048}; do
  python bench.py --r $r --no-e2e --no-cpu --no-offline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($r, round(d['value'],1), round(d['roofline']['frac'],4))"
done
