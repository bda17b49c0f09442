cd $GRAFT_REPO_ROOT
python tools/bench_lu.py 4641 10000 20890
for v in lu4 lu4m; do echo $v; VB_LIB_PATH=tools/variants/$v.so python tools/bench_lu.py 4641 10000 20890; done
