cd $GRAFT_REPO_ROOT
# the whole GPU suite on the bounds-checked build (stand-in for the closed compute-sanitizer)
VB_LIB_PATH=tools/variants/dchecks.so timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -x > gpurun_out/pytest_dchecks.log 2>&1; echo "dchecks rc=$?"
tail -5 gpurun_out/pytest_dchecks.log
grep -c "VB_DCHECK failed" gpurun_out/pytest_dchecks.log
