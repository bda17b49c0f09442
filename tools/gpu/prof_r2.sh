cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-offline --no-per-order --no-parity"
$CMD > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/prof_sweep.py --r 1024 --F 296 > gpurun_out/plain_sweep.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rom_sweep_blocked -s 2 -c 1 -o gpurun_out/r2_sweep_r1024 python tools/prof_sweep.py --r 1024 --F 296 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
python tools/prof_sweep.py --r 256 --F 592 > gpurun_out/plain_sweep256.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rom_sweep_blocked -s 2 -c 1 -o gpurun_out/r2_sweep_r256 python tools/prof_sweep.py --r 256 --F 592 > gpurun_out/ncu_full256.log 2>&1
echo "full256 rc=$?"
timeout 300 python tools/determinism_fuselage.py
