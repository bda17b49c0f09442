set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/pytest_r2a.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_r2a.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-offline > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r2a.json
