cd $GRAFT_REPO_ROOT
python tools/kron_time.py
for v in k16x8c4 k32x4c4 k16x4c8 k8x8c8; do VB_LIB_PATH=tools/variants/$v.so python tools/kron_time.py; done
