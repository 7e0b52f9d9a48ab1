# warm-push / finalize / row-table power step batch: full GPU suite, then cfg5 load steps 1..8
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/batch3
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -n 3 $O/gpu_all.log
PFB200_TRACE=1 timeout 900 python scripts/cfg5_run.py 8 S1 > $O/cfg5_trace.log 2>&1; echo "exit $?"
grep '^{"step"' $O/cfg5_trace.log | cut -c1-200
