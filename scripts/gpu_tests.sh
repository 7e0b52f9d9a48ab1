cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -30 gpurun_out/gpu_all.log
