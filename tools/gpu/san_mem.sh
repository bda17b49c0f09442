cd $GRAFT_REPO_ROOT
timeout 600 python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_memcheck.log 2>&1
echo "memcheck rc=$?"
tail -5 gpurun_out/san_memcheck.log
