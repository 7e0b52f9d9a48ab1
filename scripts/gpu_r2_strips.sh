cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/st
PFB200_TRACE=0 timeout 1200 python -m pytest tests/test_gpu_strips.py tests/test_gpu_solver.py -q -x --durations=8 > gpurun_out/st/tests.log 2>&1; echo "tests exit $?"; tail -n 15 gpurun_out/st/tests.log
