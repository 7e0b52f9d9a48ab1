# Full GPU test suite + smoke + short bench on the current tree.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/full
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/full/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -n 25 gpurun_out/full/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1; echo "smoke exit $?"; tail -n 1 gpurun_out/full/smoke.log
