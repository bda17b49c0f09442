cd $GRAFT_REPO_ROOT
python tools/prof_lu.py 10000 > gpurun_out/plain_lu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:zgetrf -s 1 -c 1 -o gpurun_out/r2_lu_n10000 python tools/prof_lu.py 10000 > gpurun_out/ncu_lu.log 2>&1
echo "ncu rc=$?"
