cd $GRAFT_REPO_ROOT
python tools/prof_cfg4.py > gpurun_out/prof_cfg4_plain.log 2>&1; echo "plain rc=$?"; cat gpurun_out/prof_cfg4_plain.log | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_cfg4_launches.csv python tools/prof_cfg4.py > gpurun_out/ncu_cfg4_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"facet_shell|zgemv_batched|hex27_helmholtz" -c 3 -o gpurun_out/r2_cfg4_kernels python tools/prof_cfg4.py > gpurun_out/ncu_cfg4_full.log 2>&1; echo "full rc=$?"
