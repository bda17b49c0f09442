# bench line (+ reference arm) + launch list + full capture of the sweep kernel (r = 1024) + offline kernels
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -1 gpurun_out/bench_default.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
tail -1 gpurun_out/bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-offline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rom_sweep_blocked --launch-skip 1 -c 1 -o gpurun_out/prof_r1024 python tools/prof_sweep.py --r 1024 --F 296 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"hex27_box_csr|spmm" --launch-skip 0 -c 4 -o gpurun_out/prof_offline python tools/prof_offline.py > gpurun_out/ncu_off.log 2>&1
ls -la gpurun_out
