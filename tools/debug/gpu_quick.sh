python -m pytest tests/test_sweep_gpu.py -x -q 2>&1 | tail -2
python tools/phase_timing.py 256 1024 2>&1 | grep -v "^r=.*F=" | tail -6
for r in 256 400 1024; do python bench.py --r $r --no-e2e --no-cpu --no-offline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($r, d[\"value\"], d[\"roofline\"][\"frac\"])"; done
