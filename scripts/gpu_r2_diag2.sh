# cfg5 load steps 1..10 with the solver trace: phase-field MG iterations per Newton solve around
# load step 8, where the load step time doubles (bench per_step_ms 1.38 s -> 3.1 s)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/diag2
mkdir -p $O
PFB200_TRACE=1 timeout 900 python scripts/cfg5_run.py 10 S1 > $O/cfg5_trace.log 2>&1; echo "exit $?"
grep '^{"step"' $O/cfg5_trace.log | cut -c1-400
grep -c "over budget" $O/cfg5_trace.log
