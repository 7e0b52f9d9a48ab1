# Gated phase-field solves by the scalar multigrid PCG (probe inside): parity tests, then cfg5
# load steps 1..10 (step 8 onwards ran ~900 Jacobi-PCG iterations per load step before).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/gated
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_mg.py tests/test_gpu_solver.py -m gpu -q -x -k "gated or spd_predicate or phase_field_mg" > $O/tests.log 2>&1; echo "tests exit $?"; tail -n 5 $O/tests.log
PFB200_TRACE=1 timeout 900 python scripts/cfg5_run.py 10 S1 > $O/cfg5_trace.log 2>&1; echo "exit $?"
grep '^{"step"' $O/cfg5_trace.log | cut -c1-330
grep "gated 1\|undecided" $O/cfg5_trace.log | sort | uniq -c | head
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -n 3 $O/gpu_all.log
