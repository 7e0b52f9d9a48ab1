# Prolongation row cache in the fine smoothing marches: kernel timings, cfg5 steps, MG tests.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/m4
timeout 600 python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/m4/prof.log 2>&1; echo "prof exit $?"; tail -n 1 gpurun_out/m4/prof.log
PFB200_TRACE=1 timeout 600 python scripts/cfg5_run.py 4 S1 > gpurun_out/m4/cfg5.log 2>&1; echo "cfg5 exit $?"; grep '^{' gpurun_out/m4/cfg5.log
timeout 1200 python -m pytest tests/test_gpu_mg.py tests/test_gpu_solver.py tests/test_bar.py tests/test_spec_properties.py -q -x > gpurun_out/m4/tests.log 2>&1; echo "tests exit $?"; tail -n 3 gpurun_out/m4/tests.log
