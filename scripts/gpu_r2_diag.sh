cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/dg
timeout 900 python -m pytest tests/test_gpu_strips.py -q -x --durations=8 > gpurun_out/dg/strips.log 2>&1; echo "strips exit $?"; tail -n 14 gpurun_out/dg/strips.log
