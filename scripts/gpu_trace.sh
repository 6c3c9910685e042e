cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in ${1:-2}; do
FFST_VERBOSE=1 timeout 300 python scripts/trace_run.py $c > gpurun_out/trace_c$c.log 2>&1; echo "trace c$c exit $?"; cat gpurun_out/trace_c$c.log | tail -16
done
