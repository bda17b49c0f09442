cd $GRAFT_REPO_ROOT
python tools/sweep_rates.py
for v in skinny3m deep512 deep4_1024 deep4_2048; do VB_LIB_PATH=tools/variants/$v.so python tools/sweep_rates.py; done
python tools/sweep_rates.py
